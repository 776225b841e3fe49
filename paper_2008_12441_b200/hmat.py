"""Thin Python binding of libhmat.so (include/hmat.h): argument marshalling only.

Every step of y = Hx runs in the library's sm_100a kernels; this module only
converts numpy arrays / torch tensors to pointers and raises on a non-zero
status.  The functions carry the C names.  There is no CPU fallback: if the
shared library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HMAT_LIB_AB") or os.path.join(_HERE, "libhmat.so")  # (A/B experiments: another build)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                      "there is no fallback path")

_lib = ctypes.CDLL(LIB_PATH)

HMAT_OK, HMAT_ERR_INVALID, HMAT_ERR_NOMEM, HMAT_ERR_CUDA, HMAT_ERR_NCCL, HMAT_ERR_UNSUPPORTED = 0, -1, -2, -3, -4, -5
HMAT_NUM_PHASES = 4
HMAT_EXCHANGE_NCCL, HMAT_EXCHANGE_EXTERNAL, HMAT_EXCHANGE_PEER, HMAT_EXCHANGE_TREE = 0, 1, 2, 3
PHASES = ("project", "exchange", "expand", "copies")

# Every symbol include/hmat.h declares (checked by tests/test_abi.py).
EXPORTS = ("hmat_create", "hmat_create_uninit", "hmat_create_strict", "hmat_create_standard",
           "hmat_create_standard_strict",
           "hmat_create_standard_uninit", "hmat_panel", "hmat_matvec", "hmat_gemv",
           "hmat_exchange_size", "hmat_project", "hmat_expand", "hmat_matvec_parts", "hmat_destroy",
           "hmat_last_error", "hmat_num_points", "hmat_local_rows", "hmat_set_stream", "hmat_nccl_unique_id",
           "hmat_nccl_selftest",
           "hmat_profile", "hmat_profile_read", "hmat_launches_per_matvec", "hmat_plan_query",
           "hmat_peer_export", "hmat_peer_import", "hmat_peer_connect_local", "hmat_cta_trace",
           "hmat_cta_trace_read", "hmat_std_exchange_query", "hmat_set_host_async", "hmat_synchronize",
           "hmat_comm_info", "hmat_exchange_size_op", "hmat_project_op", "hmat_expand_op")


class hmat_std_exchange_t(ctypes.Structure):
    _fields_ = [("E", ctypes.c_int64), ("Hn", ctypes.c_int64), ("bpad", ctypes.c_int), ("M", ctypes.c_int),
                ("src_off", ctypes.c_int64 * 64), ("zt_row_offset", ctypes.c_int64 * 64),
                ("src_entry", ctypes.c_void_p), ("src_entry_cap", ctypes.c_int64), ("n_src_entry", ctypes.c_int64),
                ("unpack", ctypes.c_void_p), ("unpack_cap", ctypes.c_int64), ("n_unpack", ctypes.c_int64),
                ("pack", ctypes.c_void_p), ("pack_cap", ctypes.c_int64), ("n_pack", ctypes.c_int64),
                ("halo_of", ctypes.c_void_p), ("halo_of_cap", ctypes.c_int64), ("n_halo_of", ctypes.c_int64),
                ("Hp", ctypes.c_int64),
                ("tpack", ctypes.c_void_p), ("tpack_cap", ctypes.c_int64), ("n_tpack", ctypes.c_int64),
                ("tadd_leaf", ctypes.c_void_p), ("tadd_leaf_cap", ctypes.c_int64), ("n_tadd_leaf", ctypes.c_int64),
                ("tadd_off", ctypes.c_void_p), ("tadd_off_cap", ctypes.c_int64), ("n_tadd_off", ctypes.c_int64),
                ("tadd_pair", ctypes.c_void_p), ("tadd_pair_cap", ctypes.c_int64), ("n_tadd_pair", ctypes.c_int64)]


class HMatError(RuntimeError):
    def __init__(self, status: int, func: str, msg: str):
        super().__init__(f"{func} failed with status {status}: {msg}")
        self.status = status


class hmat_dist_t(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int), ("rank", ctypes.c_int), ("nccl_unique_id", ctypes.c_void_p),
                ("cuda_stream", ctypes.c_void_p), ("device", ctypes.c_int), ("exchange", ctypes.c_int)]


class hmat_plan_info_t(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("c", ctypes.c_int), ("W", ctypes.c_int), ("W_pitch", ctypes.c_int), ("cross_levels", ctypes.c_int),
                ("exchange_rows", ctypes.c_int64), ("level_rows_offset", ctypes.c_int64 * 64),
                ("Rp", ctypes.c_int), ("Re", ctypes.c_int), ("tpr", ctypes.c_int), ("nstage_p", ctypes.c_int),
                ("nstage_e", ctypes.c_int), ("grid_p", ctypes.c_int), ("grid_e", ctypes.c_int),
                ("smem_p", ctypes.c_int64), ("smem_e", ctypes.c_int64),
                ("max_nr", ctypes.c_int), ("dmma", ctypes.c_int), ("dmma_ok", ctypes.c_int * 4),
                ("dmma_grid_p", ctypes.c_int * 4), ("dmma_grid_e", ctypes.c_int * 4),
                ("dmma_stages_p", ctypes.c_int * 4), ("dmma_stages_e", ctypes.c_int * 4),
                ("dmma_smem_p", ctypes.c_int64 * 4), ("dmma_smem_e", ctypes.c_int64 * 4)]


_H = ctypes.c_void_p
_P = ctypes.c_void_p
_i, _i64, _u64 = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64
_sigs = {
    "hmat_create": (_i, [_i, _i, _i, _i, _P, _P, _P, _P, ctypes.POINTER(_H)]),
    "hmat_create_uninit": (_i, [_i, _i, _i, _i, _P, ctypes.POINTER(_H)]),
    "hmat_panel": (_i, [_H, _i, _i, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                        ctypes.POINTER(_i64)]),
    "hmat_matvec": (_i, [_H, _P, _P, _i]),
    "hmat_gemv": (_i, [_H, _i, ctypes.c_double, _P, ctypes.c_double, _P, _i]),
    "hmat_create_strict": (_i, [_i, _i, _i, _i, _P, _P, _P, _P, ctypes.POINTER(_H)]),
    "hmat_create_standard": (_i, [_i, _i, _i, _i, _P, _P, _P, _P, ctypes.POINTER(_H)]),
    "hmat_create_standard_strict": (_i, [_i, _i, _i, _i, _P, _P, _P, _P, ctypes.POINTER(_H)]),
    "hmat_create_standard_uninit": (_i, [_i, _i, _i, _i, _P, ctypes.POINTER(_H)]),
    "hmat_exchange_size": (_i, [_H, _i, ctypes.POINTER(_i64)]),
    "hmat_project": (_i, [_H, _P, _i, _P]),
    "hmat_expand": (_i, [_H, _P, _P, _P, _i]),
    "hmat_matvec_parts": (_i, [_H, _P, _P, _i, _u64, _i]),
    "hmat_destroy": (_i, [_H]),
    "hmat_last_error": (ctypes.c_char_p, []),
    "hmat_num_points": (_i64, [_H]),
    "hmat_local_rows": (_i, [_H, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "hmat_set_stream": (_i, [_H, _P]),
    "hmat_nccl_unique_id": (_i, [_P]),
    "hmat_nccl_selftest": (_i, [_i, _i64]),
    "hmat_profile": (_i, [_H, _i]),
    "hmat_profile_read": (_i, [_H, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64)]),
    "hmat_launches_per_matvec": (_i64, [_H, _i]),
    "hmat_plan_query": (_i, [_i, _i, _i, _i, _i, _i, ctypes.POINTER(hmat_plan_info_t)]),
    "hmat_std_exchange_query": (_i, [_i, _i, _i, _i, _i, _i, ctypes.POINTER(hmat_std_exchange_t)]),
    "hmat_set_host_async": (_i, [_H, _i]),
    "hmat_synchronize": (_i, [_H]),
    "hmat_comm_info": (_i, [_H, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "hmat_exchange_size_op": (_i, [_H, _i, _i, ctypes.POINTER(_i64)]),
    "hmat_project_op": (_i, [_H, _i, _P, _i, _P]),
    "hmat_expand_op": (_i, [_H, _i, ctypes.c_double, _P, _P, ctypes.c_double, _P, _i]),
    "hmat_peer_export": (_i, [_H, _P]),
    "hmat_cta_trace": (_i, [_H, _i]),
    "hmat_cta_trace_read": (_i, [_H, _i, ctypes.POINTER(ctypes.c_int64), _i, ctypes.POINTER(ctypes.c_int)]),
    "hmat_peer_import": (_i, [_H, _P]),
    "hmat_peer_connect_local": (_i, [_H, _P]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def hmat_last_error() -> str:
    return _lib.hmat_last_error().decode()


def _check(status: int, func: str):
    if status != HMAT_OK:
        raise HMatError(status, func, hmat_last_error())


def _ptr(a):
    """Raw address of a numpy array or torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise TypeError(f"cannot take the address of {type(a)}")


def _panel_ok(a, rows: int, cols: int):
    if isinstance(a, np.ndarray):
        assert a.dtype == np.float64 and a.flags.c_contiguous and a.shape == (rows, cols), \
            f"panel must be C-contiguous float64 {(rows, cols)}, got {a.dtype} {a.shape}"
    elif hasattr(a, "data_ptr"):
        import torch
        assert a.dtype == torch.float64 and a.is_contiguous() and tuple(a.shape) == (rows, cols), \
            f"panel must be contiguous float64 {(rows, cols)}"


def _vec(a, n: int):
    """(pointer, nrhs) of an N_loc x nrhs column-major block: a 1-D array of n
    values, or a 2-D (n, nrhs) array with column-major strides."""
    if isinstance(a, np.ndarray):
        assert a.dtype == np.float64
        if a.ndim == 1:
            assert a.shape[0] == n and a.flags.c_contiguous
            return a.ctypes.data, 1
        assert a.shape[0] == n and a.flags.f_contiguous, "x/y must be (N_loc, nrhs) column-major"
        return a.ctypes.data, a.shape[1]
    import torch
    assert a.dtype == torch.float64
    if a.dim() == 1:
        assert a.shape[0] == n and a.is_contiguous()
        return a.data_ptr(), 1
    assert a.shape[0] == n and (a.shape[1] == 1 or a.stride() == (1, n)), "x/y must be (N_loc, nrhs) column-major"
    return a.data_ptr(), a.shape[1]


def _dist(nranks=1, rank=0, nccl_unique_id=None, cuda_stream=None, device=None, external_exchange=False,
          exchange=None):
    d = hmat_dist_t()
    d.nranks, d.rank = nranks, rank
    d.exchange = exchange if exchange is not None else (HMAT_EXCHANGE_EXTERNAL if external_exchange
                                                        else HMAT_EXCHANGE_NCCL)
    d._id_buf = None
    if nccl_unique_id is not None:
        buf = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
        d._id_buf = buf
        d.nccl_unique_id = ctypes.cast(buf, ctypes.c_void_p)
    d.cuda_stream = cuda_stream
    if device is None:
        import torch
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    d.device = device
    return d


def hmat_create(depth, dim, leaf_size, rank, U, V, D, dist: hmat_dist_t | None = None):
    """H from canonical panels (list of `depth` U_l, list of V_l, D), host or device."""
    Up = (ctypes.c_void_p * max(1, len(U)))(*[_ptr(u) for u in U])
    Vp = (ctypes.c_void_p * max(1, len(V)))(*[_ptr(v) for v in V])
    h = _H()
    _check(_lib.hmat_create(depth, dim, leaf_size, rank, ctypes.cast(Up, _P), ctypes.cast(Vp, _P), _ptr(D),
                            ctypes.byref(dist) if dist is not None else None, ctypes.byref(h)), "hmat_create")
    return h


def hmat_create_strict(depth, dim, leaf_size, rank, U, V, Dc, dist: hmat_dist_t | None = None):
    """Paper-strict Def 2.4 structure: U, V = depth-1 panels, Dc = N x (2^dim leaf) dense panel."""
    Up = (ctypes.c_void_p * max(1, len(U)))(*[_ptr(u) for u in U])
    Vp = (ctypes.c_void_p * max(1, len(V)))(*[_ptr(v) for v in V])
    h = _H()
    _check(_lib.hmat_create_strict(depth, dim, leaf_size, rank, ctypes.cast(Up, _P), ctypes.cast(Vp, _P), _ptr(Dc),
                                   ctypes.byref(dist) if dist is not None else None, ctypes.byref(h)),
           "hmat_create_strict")
    return h


def hmat_create_standard(depth, dim, leaf_size, rank, U, V, Dn, dist: hmat_dist_t | None = None):
    """Standard admissibility (interaction lists + near field); canonical standard panels."""
    Up = (ctypes.c_void_p * max(1, len(U)))(*[_ptr(u) for u in U])
    Vp = (ctypes.c_void_p * max(1, len(V)))(*[_ptr(v) for v in V])
    h = _H()
    _check(_lib.hmat_create_standard(depth, dim, leaf_size, rank, ctypes.cast(Up, _P), ctypes.cast(Vp, _P),
                                     _ptr(Dn), ctypes.byref(dist) if dist is not None else None, ctypes.byref(h)),
           "hmat_create_standard")
    return h


def hmat_create_standard_strict(depth, dim, leaf_size, rank, U, V, Dc, dist: hmat_dist_t | None = None):
    """Standard admissibility with Def 2.4 read literally (leaf first): U, V = depth-1
    standard panels, Dc = N x (3^dim 2^dim leaf) leaf-parent near-field panel."""
    Up = (ctypes.c_void_p * max(1, len(U)))(*[_ptr(u) for u in U])
    Vp = (ctypes.c_void_p * max(1, len(V)))(*[_ptr(v) for v in V])
    h = _H()
    _check(_lib.hmat_create_standard_strict(depth, dim, leaf_size, rank, ctypes.cast(Up, _P), ctypes.cast(Vp, _P),
                                            _ptr(Dc), ctypes.byref(dist) if dist is not None else None,
                                            ctypes.byref(h)),
           "hmat_create_standard_strict")
    return h


def hmat_create_standard_uninit(depth, dim, leaf_size, rank, dist: hmat_dist_t | None = None):
    h = _H()
    _check(_lib.hmat_create_standard_uninit(depth, dim, leaf_size, rank,
                                            ctypes.byref(dist) if dist is not None else None, ctypes.byref(h)),
           "hmat_create_standard_uninit")
    return h


def hmat_create_uninit(depth, dim, leaf_size, rank, dist: hmat_dist_t | None = None):
    h = _H()
    _check(_lib.hmat_create_uninit(depth, dim, leaf_size, rank, ctypes.byref(dist) if dist is not None else None,
                                   ctypes.byref(h)), "hmat_create_uninit")
    return h


def hmat_panel(h, kind: int, level: int):
    """(device pointer, rows, cols, ld) of panel kind 0=U_level, 1=V_level, 2=D."""
    ptr, rows, cols, ld = ctypes.c_void_p(), _i64(), _i64(), _i64()
    _check(_lib.hmat_panel(h, kind, level, ctypes.byref(ptr), ctypes.byref(rows), ctypes.byref(cols),
                           ctypes.byref(ld)), "hmat_panel")
    return ptr.value, rows.value, cols.value, ld.value


def hmat_matvec(h, x, y, nrhs: int | None = None):
    n = hmat_local_rows(h)
    n = n[1] - n[0]
    xp, kx = _vec(x, n)
    yp, ky = _vec(y, n)
    nrhs = kx if nrhs is None else nrhs
    assert kx >= nrhs and ky >= nrhs
    _check(_lib.hmat_matvec(h, xp, yp, nrhs), "hmat_matvec")


def hmat_gemv(h, trans: int, alpha: float, x, beta: float, y, nrhs: int | None = None):
    """y = alpha op(H) x + beta y, op = H (trans=0) or H^T (trans=1)."""
    n = hmat_local_rows(h)
    n = n[1] - n[0]
    xp, kx = _vec(x, n)
    yp, ky = _vec(y, n)
    nrhs = kx if nrhs is None else nrhs
    assert kx >= nrhs and ky >= nrhs
    _check(_lib.hmat_gemv(h, int(trans), float(alpha), xp, float(beta), yp, nrhs), "hmat_gemv")


def hmat_exchange_size(h, nrhs: int) -> int:
    """doubles of one pass's packed exchange buffer (0 when P = 1)."""
    cnt = _i64()
    _check(_lib.hmat_exchange_size(h, nrhs, ctypes.byref(cnt)), "hmat_exchange_size")
    return cnt.value


def hmat_project(h, x, exchange, nrhs: int | None = None):
    """Split phase 1: this rank's contributions -> exchange (device, >= exchange_size doubles)."""
    n = hmat_local_rows(h)
    n = n[1] - n[0]
    xp, kx = _vec(x, n)
    nrhs = kx if nrhs is None else nrhs
    _check(_lib.hmat_project(h, xp, nrhs, _ptr(exchange)), "hmat_project")


def hmat_expand(h, x, exchange, y, nrhs: int | None = None):
    """Split phase 3: y = H x from the exchange buffer summed over all ranks."""
    n = hmat_local_rows(h)
    n = n[1] - n[0]
    xp, kx = _vec(x, n)
    yp, ky = _vec(y, n)
    nrhs = kx if nrhs is None else nrhs
    _check(_lib.hmat_expand(h, xp, _ptr(exchange), yp, nrhs), "hmat_expand")


def hmat_exchange_size_op(h, trans: int, nrhs: int) -> int:
    """doubles of one pass's packed exchange buffer for op(H) (0 when P = 1)."""
    cnt = _i64()
    _check(_lib.hmat_exchange_size_op(h, int(trans), nrhs, ctypes.byref(cnt)), "hmat_exchange_size_op")
    return cnt.value


def hmat_project_op(h, trans: int, x, exchange, nrhs: int | None = None):
    """Split phase 1 of y = alpha op(H) x + beta y."""
    n = hmat_local_rows(h)
    n = n[1] - n[0]
    xp, kx = _vec(x, n)
    nrhs = kx if nrhs is None else nrhs
    _check(_lib.hmat_project_op(h, int(trans), xp, nrhs, _ptr(exchange)), "hmat_project_op")


def hmat_expand_op(h, trans: int, alpha: float, x, exchange, beta: float, y, nrhs: int | None = None):
    """Split phase 3: y = alpha op(H) x + beta y from the exchange summed over all ranks."""
    n = hmat_local_rows(h)
    n = n[1] - n[0]
    xp, kx = _vec(x, n)
    yp, ky = _vec(y, n)
    nrhs = kx if nrhs is None else nrhs
    _check(_lib.hmat_expand_op(h, int(trans), float(alpha), xp, _ptr(exchange), float(beta), yp, nrhs),
           "hmat_expand_op")


def hmat_matvec_parts(h, x, y, level_mask: int, dense: bool, nrhs: int | None = None):
    n = hmat_local_rows(h)
    n = n[1] - n[0]
    xp, kx = _vec(x, n)
    yp, ky = _vec(y, n)
    nrhs = kx if nrhs is None else nrhs
    _check(_lib.hmat_matvec_parts(h, xp, yp, nrhs, level_mask & ((1 << 64) - 1), int(bool(dense))),
           "hmat_matvec_parts")


def hmat_destroy(h):
    _check(_lib.hmat_destroy(h), "hmat_destroy")


def hmat_num_points(h) -> int:
    return _lib.hmat_num_points(h)


def hmat_local_rows(h):
    b, e = _i64(), _i64()
    _check(_lib.hmat_local_rows(h, ctypes.byref(b), ctypes.byref(e)), "hmat_local_rows")
    return b.value, e.value


def hmat_set_stream(h, stream: int):
    _check(_lib.hmat_set_stream(h, stream), "hmat_set_stream")


def hmat_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.hmat_nccl_unique_id(ctypes.cast(buf, _P)), "hmat_nccl_unique_id")
    return buf.raw


def hmat_nccl_selftest(device: int = 0, count: int = 4096):
    _check(_lib.hmat_nccl_selftest(device, count), "hmat_nccl_selftest")


def hmat_profile(h, enable: bool):
    _check(_lib.hmat_profile(h, int(bool(enable))), "hmat_profile")


def hmat_profile_read(h):
    """{phase: (milliseconds, launches)} accumulated since the last read."""
    ms = (ctypes.c_double * HMAT_NUM_PHASES)()
    nl = (_i64 * HMAT_NUM_PHASES)()
    _check(_lib.hmat_profile_read(h, ms, nl), "hmat_profile_read")
    return {PHASES[i]: (ms[i], nl[i]) for i in range(HMAT_NUM_PHASES)}


def hmat_launches_per_matvec(h, nrhs: int) -> int:
    return _lib.hmat_launches_per_matvec(h, nrhs)


def hmat_plan_query(depth, dim, leaf_size, rank, nranks=1, rank_id=0) -> hmat_plan_info_t:
    info = hmat_plan_info_t()
    _check(_lib.hmat_plan_query(depth, dim, leaf_size, rank, nranks, rank_id, ctypes.byref(info)),
           "hmat_plan_query")
    return info


def hmat_set_host_async(h, enable: bool = True) -> None:
    """Asynchronous host-pointer mode (include/hmat.h): host-pointer matvecs
    return once enqueued; keep x / y valid until hmat_synchronize(h)."""
    _check(_lib.hmat_set_host_async(h, 1 if enable else 0), "hmat_set_host_async")


def hmat_synchronize(h) -> None:
    _check(_lib.hmat_synchronize(h), "hmat_synchronize")


def hmat_comm_info(h):
    """(nranks, rank) of the communicator h exchanges over (NCCL's own view for
    the NCCL / TREE exchanges); raises on a pending asynchronous exchange error."""
    n, r = ctypes.c_int(), ctypes.c_int()
    _check(_lib.hmat_comm_info(h, ctypes.byref(n), ctypes.byref(r)), "hmat_comm_info")
    return n.value, r.value


def hmat_std_exchange_query(depth, dim, leaf_size, rank, nranks, rank_id) -> dict:
    """The packed cross-rank exchange of one rank of a standard-admissibility
    operator (include/hmat.h): counts, offsets and this rank's tables (numpy)."""
    import numpy as np
    q = hmat_std_exchange_t()
    _check(_lib.hmat_std_exchange_query(depth, dim, leaf_size, rank, nranks, rank_id, ctypes.byref(q)),
           "hmat_std_exchange_query")
    src = np.zeros(max(1, q.n_src_entry), dtype=np.int32)
    unp = np.zeros(max(1, 2 * (q.n_unpack // 2)), dtype=np.int64)
    pk = np.zeros(max(1, q.n_pack), dtype=np.int64)
    ho = np.zeros(max(1, q.n_halo_of), dtype=np.int32)
    q.src_entry, q.src_entry_cap = src.ctypes.data, src.size
    q.unpack, q.unpack_cap = unp.ctypes.data, unp.size
    q.pack, q.pack_cap = pk.ctypes.data, pk.size
    q.halo_of, q.halo_of_cap = ho.ctypes.data, ho.size
    tp = np.zeros(max(1, q.n_tpack), dtype=np.int64)
    tl = np.zeros(max(1, q.n_tadd_leaf), dtype=np.int64)
    to = np.zeros(max(1, q.n_tadd_off), dtype=np.int64)
    tq = np.zeros(max(1, q.n_tadd_pair), dtype=np.int64)
    q.tpack, q.tpack_cap = tp.ctypes.data, tp.size
    q.tadd_leaf, q.tadd_leaf_cap = tl.ctypes.data, tl.size
    q.tadd_off, q.tadd_off_cap = to.ctypes.data, to.size
    q.tadd_pair, q.tadd_pair_cap = tq.ctypes.data, tq.size
    _check(_lib.hmat_std_exchange_query(depth, dim, leaf_size, rank, nranks, rank_id, ctypes.byref(q)),
           "hmat_std_exchange_query")
    return {"E": q.E, "Hn": q.Hn, "bpad": q.bpad, "M": q.M, "src_off": list(q.src_off)[:depth + 1],
            "zt_row_offset": list(q.zt_row_offset)[:depth + 1], "src_entry": src[:q.n_src_entry],
            "unpack": unp[:q.n_unpack].reshape(-1, 2), "pack": pk[:q.n_pack].reshape(-1, 2),
            "halo_of": ho[:q.n_halo_of], "Hp": q.Hp, "tpack": tp[:q.n_tpack].reshape(-1, 3),
            "tadd_leaf": tl[:q.n_tadd_leaf], "tadd_off": to[:q.n_tadd_off], "tadd_pair": tq[:q.n_tadd_pair]}


class HMatrix:
    """Owning convenience wrapper around an hmat_t handle."""

    def __init__(self, depth, dim, leaf_size, rank, U=None, V=None, D=None, dist=None):
        self.depth, self.dim, self.leaf_size, self.rank = depth, dim, leaf_size, rank
        self._dist = dist
        if D is None:
            self.h = hmat_create_uninit(depth, dim, leaf_size, rank, dist)
        else:
            self.h = hmat_create(depth, dim, leaf_size, rank, U, V, D, dist)

    @property
    def rows(self):
        return hmat_local_rows(self.h)

    def matvec(self, x, y, nrhs=None):
        hmat_matvec(self.h, x, y, nrhs)
        return y

    def parts(self, x, y, level_mask, dense, nrhs=None):
        hmat_matvec_parts(self.h, x, y, level_mask, dense, nrhs)
        return y

    def close(self):
        if self.h is not None and self.h.value:
            hmat_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hmat_peer_export(h) -> bytes:
    """64-byte CUDA IPC handle of this rank's peer-exchange mailbox."""
    buf = ctypes.create_string_buffer(64)
    _check(_lib.hmat_peer_export(h, ctypes.cast(buf, _P)), "hmat_peer_export")
    return buf.raw


def hmat_peer_import(h, handles):
    """handles: the P ranks' 64-byte handles in rank order."""
    blob = ctypes.create_string_buffer(b"".join(bytes(x) for x in handles), 64 * len(handles))
    _check(_lib.hmat_peer_import(h, ctypes.cast(blob, _P)), "hmat_peer_import")


def hmat_peer_connect_local(h, ranks):
    """connect the mailboxes of P handles of this process (rank order)."""
    arr = (ctypes.c_void_p * len(ranks))(*[r.value for r in ranks])
    _check(_lib.hmat_peer_connect_local(h, ctypes.cast(arr, _P)), "hmat_peer_connect_local")


def hmat_cta_trace(h, enable=True):
    _check(_lib.hmat_cta_trace(h, int(bool(enable))), "hmat_cta_trace")


def hmat_cta_trace_read(h, kernel, max_ctas=8192):
    """[(start_ns, end_ns, sm_id)] per CTA of the last project (0) / expand (1) launch."""
    buf = (ctypes.c_int64 * (3 * max_ctas))()
    n = ctypes.c_int(0)
    _check(_lib.hmat_cta_trace_read(h, kernel, buf, max_ctas, ctypes.byref(n)), "hmat_cta_trace_read")
    return [(buf[3 * b], buf[3 * b + 1], buf[3 * b + 2]) for b in range(n.value)]
