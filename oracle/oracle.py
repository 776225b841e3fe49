"""CPU oracle for y = Hx (weak admissibility) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  It wraps oracle/liboracle.so (plain C,
fp64, -ffp-contract=off), which shares no code with the CUDA path.  See the
header of oracle/hmat_oracle.c for the paper passages each function follows.

Every function is pinned by tests/test_oracle_pins.py (brute force, closed
forms, special cases, the paper's block count); see DESIGN.md §5.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)


def _load():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.oracle_sibling.restype = ctypes.c_int64
        lib.oracle_sibling.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int]
        lib.oracle_slot.restype = ctypes.c_int
        lib.oracle_slot.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64]
        lib.oracle_block_census.restype = None
        lib.oracle_block_census.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.POINTER(ctypes.c_int64)] * 3
        lib.oracle_cover_count.restype = None
        lib.oracle_cover_count.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        pp = ctypes.POINTER(_dp)
        lib.oracle_matvec_masked.restype = None
        lib.oracle_matvec_masked.argtypes = [ctypes.c_int] * 4 + [pp, pp, ctypes.c_void_p, ctypes.c_void_p,
                                                                 ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64,
                                                                 ctypes.c_int]
        lib.oracle_assemble.restype = None
        lib.oracle_assemble.argtypes = [ctypes.c_int] * 4 + [pp, pp, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_block_census_strict.restype = None
        lib.oracle_block_census_strict.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.POINTER(ctypes.c_int64)] * 3
        lib.oracle_cover_count_v.restype = None
        lib.oracle_cover_count_v.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p]
        lib.oracle_assemble_v.restype = None
        lib.oracle_assemble_v.argtypes = [ctypes.c_int] * 5 + [pp, pp, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_matvec_t.restype = None
        lib.oracle_matvec_t.argtypes = [ctypes.c_int] * 4 + [pp, pp, ctypes.c_void_p, ctypes.c_void_p,
                                                             ctypes.c_void_p, ctypes.c_int]
        lib.oracle_matvec_strict.restype = None
        lib.oracle_matvec_strict.argtypes = [ctypes.c_int] * 4 + [pp, pp, ctypes.c_void_p, ctypes.c_void_p,
                                                                  ctypes.c_void_p, ctypes.c_int]
        lib.oracle_dense_matvec.restype = None
        lib.oracle_dense_matvec.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_int]
        lib.oracle_rows_generated.restype = None
        lib.oracle_rows_generated.argtypes = [ctypes.c_int] * 4 + [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                                                                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_matvec_rows_par.restype = None
        lib.oracle_matvec_rows_par.argtypes = [ctypes.c_int] * 4 + [pp, pp, ctypes.c_void_p, ctypes.c_uint64,
                                                                    ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                                                    ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                                                    ctypes.c_uint64, ctypes.c_int, ctypes.c_int]
        _lib = lib
    return _lib


def host_threads() -> int:
    """Host cores this process may use (cgroup / taskset aware)."""
    return len(os.sched_getaffinity(0))


def _c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _panel_ptrs(panels):
    arrs = [_c(p) for p in panels]
    ptrs = (_dp * max(1, len(arrs)))(*[a.ctypes.data_as(_dp) for a in arrs])
    return arrs, ptrs


def _colmajor(x: np.ndarray) -> np.ndarray:
    """x as an (N, nrhs) Fortran-order float64 array (column-major, ld = N)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    return np.asfortranarray(x)


def sibling(c: int, t: int, q: int) -> int:
    return _load().oracle_sibling(c, t, q)


def slot(c: int, t: int, s: int) -> int:
    return _load().oracle_slot(c, t, s)


def block_census(d: int, L: int):
    """(#low-rank blocks, #dense blocks, #low-rank blocks at level 1), counted by
    walking Def 2.4's recursion."""
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _load().oracle_block_census(d, L, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    return a.value, b.value, c.value


def cover_count(d: int, L: int, b: int) -> np.ndarray:
    N = b * (1 << d) ** L
    out = np.zeros((N, N), dtype=np.int32)
    _load().oracle_cover_count(d, L, b, out.ctypes.data)
    return out


def matvec(d: int, L: int, b: int, r: int, U, V, D, x, level_mask: int = (1 << 64) - 1,
           dense: bool = True) -> np.ndarray:
    """y = H x by the block loop of eq:hmat-vec-add.  x: (N,) or (N, nrhs)."""
    xc = _colmajor(x)
    N, nrhs = xc.shape
    y = np.zeros((N, nrhs), dtype=np.float64, order="F")
    ua, up = _panel_ptrs(U)
    va, vp = _panel_ptrs(V)
    Dc = _c(D)
    _load().oracle_matvec_masked(d, L, b, r, up, vp, Dc.ctypes.data, xc.ctypes.data, y.ctypes.data, nrhs,
                                 level_mask & ((1 << 64) - 1), int(dense))
    return y[:, 0] if np.ndim(x) == 1 else y


def assemble(d: int, L: int, b: int, r: int, U, V, D) -> np.ndarray:
    N = b * (1 << d) ** L
    A = np.zeros((N, N), dtype=np.float64)
    ua, up = _panel_ptrs(U)
    va, vp = _panel_ptrs(V)
    Dc = _c(D)
    _load().oracle_assemble(d, L, b, r, up, vp, Dc.ctypes.data, A.ctypes.data)
    return A


def dense_matvec(A: np.ndarray, x) -> np.ndarray:
    """y = A x by the definition (plain double loop in C)."""
    Ac = _c(A)
    xc = _colmajor(x)
    N, nrhs = xc.shape
    y = np.zeros((N, nrhs), dtype=np.float64, order="F")
    _load().oracle_dense_matvec(N, Ac.ctypes.data, xc.ctypes.data, y.ctypes.data, nrhs)
    return y[:, 0] if np.ndim(x) == 1 else y


def rows_generated(cfg, x, rows) -> np.ndarray:
    """y[rows, :] for the seeded synthetic H-matrix of `cfg` (gen/hgen.h), factor
    entries generated on demand; x: (N,) or (N, nrhs) host array."""
    xc = _colmajor(x)
    N, nrhs = xc.shape
    assert N == cfg.N
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((len(rows), nrhs), dtype=np.float64, order="F")
    _load().oracle_rows_generated(cfg.d, cfg.L, cfg.b, cfg.r, cfg.seed, xc.ctypes.data, nrhs, len(rows),
                                  rows.ctypes.data, out.ctypes.data)
    return out[:, 0] if np.ndim(x) == 1 else out


def matvec_par(d: int, L: int, b: int, r: int, U, V, D, x, threads: int | None = None, row_begin: int = 0,
               row_end: int | None = None, level_mask: int = (1 << 64) - 1, dense: bool = True) -> np.ndarray:
    """Rows [row_begin, row_end) of y = H x: the block loop of `matvec` on all
    host cores (bit-identical to it for any thread count, oracle_matvec_rows_par)."""
    xc = _colmajor(x)
    N, nrhs = xc.shape
    r1 = N if row_end is None else row_end
    y = np.zeros((r1 - row_begin, nrhs), dtype=np.float64, order="F")
    ua, up = _panel_ptrs(U)
    va, vp = _panel_ptrs(V)
    Dc = _c(D)
    _load().oracle_matvec_rows_par(d, L, b, r, up, vp, Dc.ctypes.data, 0, xc.ctypes.data, nrhs, row_begin, r1,
                                   y.ctypes.data, max(1, r1 - row_begin), level_mask & ((1 << 64) - 1), int(dense),
                                   threads or host_threads())
    return y[:, 0] if np.ndim(x) == 1 else y


def matvec_generated(cfg, x, row_begin: int = 0, row_end: int | None = None, threads: int | None = None,
                     level_mask: int = (1 << 64) - 1, dense: bool = True) -> np.ndarray:
    """Rows [row_begin, row_end) of y = H x for the seeded synthetic H-matrix of
    `cfg` (gen/hgen.h), every factor entry generated on demand (no factor memory:
    full-size BASELINE operators on the host), all host cores; bit-identical to
    `matvec` on the panels of hgen.inputs(cfg).  x: (N,) or (N, nrhs), full."""
    xc = _colmajor(x)
    N, nrhs = xc.shape
    assert N == cfg.N
    r1 = N if row_end is None else row_end
    y = np.zeros((r1 - row_begin, nrhs), dtype=np.float64, order="F")
    null = ctypes.POINTER(_dp)()
    _load().oracle_matvec_rows_par(cfg.d, cfg.L, cfg.b, cfg.r, null, null, None, cfg.seed, xc.ctypes.data, nrhs,
                                   row_begin, r1, y.ctypes.data, max(1, r1 - row_begin),
                                   level_mask & ((1 << 64) - 1), int(dense), threads or host_threads())
    return y[:, 0] if np.ndim(x) == 1 else y


def block_census_strict(d: int, L: int):
    """Block counts of the paper-strict reading of Def 2.4 (leaves checked first)."""
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _load().oracle_block_census_strict(d, L, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    return a.value, b.value, c.value


def cover_count_strict(d: int, L: int, b: int) -> np.ndarray:
    N = b * (1 << d) ** L
    out = np.zeros((N, N), dtype=np.int32)
    _load().oracle_cover_count_v(1, d, L, b, out.ctypes.data)
    return out


def assemble_strict(d: int, L: int, b: int, r: int, U, V, Dc) -> np.ndarray:
    """Strict structure: U, V = levels 1..L-1, Dc = N x (2^d b) leaf-parent dense panel."""
    N = b * (1 << d) ** L
    A = np.zeros((N, N), dtype=np.float64)
    ua, up = _panel_ptrs(U)
    va, vp = _panel_ptrs(V)
    Dc = _c(Dc)
    _load().oracle_assemble_v(1, d, L, b, r, up, vp, Dc.ctypes.data, A.ctypes.data)
    return A


def _mv(fn, d, L, b, r, U, V, D, x):
    xc = _colmajor(x)
    N, nrhs = xc.shape
    y = np.zeros((N, nrhs), dtype=np.float64, order="F")
    ua, up = _panel_ptrs(U)
    va, vp = _panel_ptrs(V)
    Dc = _c(D)
    fn(d, L, b, r, up, vp, Dc.ctypes.data, xc.ctypes.data, y.ctypes.data, nrhs)
    return y[:, 0] if np.ndim(x) == 1 else y


def matvec_t(d: int, L: int, b: int, r: int, U, V, D, x) -> np.ndarray:
    """y = H^T x by the transposed block loop."""
    return _mv(_load().oracle_matvec_t, d, L, b, r, U, V, D, x)


def matvec_strict(d: int, L: int, b: int, r: int, U, V, Dc, x) -> np.ndarray:
    """y = H x for the paper-strict structure (U, V levels 1..L-1, leaf-parent dense panel)."""
    return _mv(_load().oracle_matvec_strict, d, L, b, r, U, V, Dc, x)


# -- standard admissibility ------------------------------------------

def _std_lib():
    lib = _load()
    if not getattr(lib, "_std_ready", False):
        pp = ctypes.POINTER(_dp)
        lib.oracle_std_slots.restype = ctypes.c_int
        lib.oracle_std_slots.argtypes = [ctypes.c_int]
        lib.oracle_std_slot.restype = ctypes.c_int
        lib.oracle_std_slot.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64]
        lib.oracle_std_census.restype = None
        lib.oracle_std_census.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64] + \
            [ctypes.POINTER(ctypes.c_int64)] * 3
        lib.oracle_std_cover_count.restype = None
        lib.oracle_std_cover_count.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p]
        lib.oracle_std_assemble.restype = None
        lib.oracle_std_assemble.argtypes = [ctypes.c_int] * 4 + [pp, pp, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_std_matvec.restype = None
        lib.oracle_std_matvec.argtypes = [ctypes.c_int] * 4 + [pp, pp, ctypes.c_void_p, ctypes.c_void_p,
                                                               ctypes.c_void_p, ctypes.c_int]
        lib.oracle_std_matvec_t.restype = None
        lib.oracle_std_matvec_t.argtypes = lib.oracle_std_matvec.argtypes
        lib.oracle_std_rows_generated.restype = None
        lib.oracle_std_rows_generated.argtypes = lib.oracle_rows_generated.argtypes
        lib.oracle_std_census_strict.restype = None
        lib.oracle_std_census_strict.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.POINTER(ctypes.c_int64)] * 2
        lib.oracle_std_cover_count_strict.restype = None
        lib.oracle_std_cover_count_strict.argtypes = lib.oracle_std_cover_count.argtypes
        lib.oracle_std_assemble_strict.restype = None
        lib.oracle_std_assemble_strict.argtypes = lib.oracle_std_assemble.argtypes
        lib.oracle_std_matvec_strict.restype = None
        lib.oracle_std_matvec_strict.argtypes = lib.oracle_std_matvec.argtypes
        lib._std_ready = True
    return lib


def std_slots(d: int) -> int:
    """M = 6^d - 3^d interaction slots per node."""
    return _std_lib().oracle_std_slots(d)


def std_slot(d: int, level: int, t: int, s: int) -> int:
    return _std_lib().oracle_std_slot(d, level, t, s)


def std_census(d: int, L: int, level: int = 0, target: int = -1):
    """(#low-rank, #dense, #low-rank blocks of `target` at `level`) by walking
    Def 2.4 with standard admissibility."""
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _std_lib().oracle_std_census(d, L, level, target, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    return a.value, b.value, c.value


def std_cover_count(d: int, L: int, b: int) -> np.ndarray:
    N = b * (1 << d) ** L
    out = np.zeros((N, N), dtype=np.int32)
    _std_lib().oracle_std_cover_count(d, L, b, out.ctypes.data)
    return out


def std_assemble(d: int, L: int, b: int, r: int, U, V, Dn) -> np.ndarray:
    N = b * (1 << d) ** L
    A = np.zeros((N, N), dtype=np.float64)
    ua, up = _panel_ptrs(U)
    va, vp = _panel_ptrs(V)
    Dn = _c(Dn)
    _std_lib().oracle_std_assemble(d, L, b, r, up, vp, Dn.ctypes.data, A.ctypes.data)
    return A


def std_matvec(d: int, L: int, b: int, r: int, U, V, Dn, x) -> np.ndarray:
    _std_lib()
    return _mv(_load().oracle_std_matvec, d, L, b, r, U, V, Dn, x)


def std_matvec_t(d: int, L: int, b: int, r: int, U, V, Dn, x) -> np.ndarray:
    """y = H^T x by the transposed standard-admissibility block loop."""
    _std_lib()
    return _mv(_load().oracle_std_matvec_t, d, L, b, r, U, V, Dn, x)


def std_census_strict(d: int, L: int):
    """(#low-rank, #dense) blocks of the literal-order (leaf-first) standard structure."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _std_lib().oracle_std_census_strict(d, L, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def std_cover_count_strict(d: int, L: int, b: int) -> np.ndarray:
    N = b * (1 << d) ** L
    out = np.zeros((N, N), dtype=np.int32)
    _std_lib().oracle_std_cover_count_strict(d, L, b, out.ctypes.data)
    return out


def std_assemble_strict(d: int, L: int, b: int, r: int, U, V, Dc) -> np.ndarray:
    N = b * (1 << d) ** L
    A = np.zeros((N, N), dtype=np.float64)
    ua, up = _panel_ptrs(U)
    va, vp = _panel_ptrs(V)
    Dc = _c(Dc)
    _std_lib().oracle_std_assemble_strict(d, L, b, r, up, vp, Dc.ctypes.data, A.ctypes.data)
    return A


def std_matvec_strict(d: int, L: int, b: int, r: int, U, V, Dc, x) -> np.ndarray:
    """y = H x for the literal-order (leaf-first) standard structure."""
    _std_lib()
    return _mv(_load().oracle_std_matvec_strict, d, L, b, r, U, V, Dc, x)


def std_rows_generated(cfg, x, rows) -> np.ndarray:
    """y[rows, :] of the seeded standard-admissibility operator of `cfg` (factor
    entries generated on demand, blocks found by the Def 2.4 recursion
    restricted to each row); x: (N,) or (N, nrhs) host array."""
    lib = _std_lib()
    xc = _colmajor(x)
    N, nrhs = xc.shape
    assert N == cfg.N and cfg.adm == 1
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((len(rows), nrhs), dtype=np.float64, order="F")
    lib.oracle_std_rows_generated(cfg.d, cfg.L, cfg.b, cfg.r, cfg.seed, xc.ctypes.data, nrhs, len(rows),
                                  rows.ctypes.data, out.ctypes.data)
    return out[:, 0] if np.ndim(x) == 1 else out
