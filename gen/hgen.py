"""Seeded synthetic inputs (TEST/BENCH INFRASTRUCTURE; no H-matvec arithmetic).

Python face of gen/hgen.h: the configuration table C1..C5 of BASELINE.json and
fillers for the canonical panels.  The paper's benchmark
matrices are "filled ... by random numbers" with random input vectors
(PAPER.md:1121-1125); BASELINE.json fixes the distributions:
U, V ~ N(0,1)/sqrt(block rows), D ~ N(0,1)/8, x ~ U[-1,1].

The host filler (libhgen.so) and the device filler (libhgen_dev.so) produce
bit-identical values (integer hashing + correctly rounded +,-,*,/,sqrt only).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

TAG_U, TAG_V, TAG_D, TAG_X = 1, 2, 3, 4
SEED_BASE = 200812441  # seed = SEED_BASE + config index (1..5)


@dataclass(frozen=True)
class HConfig:
    """One H-matrix workload: dimension d, depth L, leaf size b, rank r."""
    name: str
    d: int
    L: int
    b: int
    r: int
    nrhs: int = 1
    seed: int = SEED_BASE
    adm: int = 0  # 0 = weak admissibility, 1 = standard admissibility

    @property
    def c(self) -> int:
        return 1 << self.d

    @property
    def N(self) -> int:
        return self.b * self.c ** self.L

    @property
    def slots(self) -> int:
        """low-rank slots per node: 2^d - 1 siblings (weak) or 6^d - 3^d (standard)."""
        return self.c - 1 if self.adm == 0 else 6 ** self.d - 3 ** self.d

    @property
    def W(self) -> int:
        return self.slots * self.r

    @property
    def dcols(self) -> int:
        """columns of the dense panel: b (leaf diagonal) or 3^d b (near field)."""
        return self.b if self.adm == 0 else 3 ** self.d * self.b

    def m(self, level: int) -> int:
        """Rows of a level-`level` node, m_l = N / c^l."""
        return self.N // self.c ** level

    def lowrank_scale(self, level: int) -> float:
        """1/sqrt(block rows) for U_l and V_l (BASELINE.json; R8)."""
        return 1.0 / math.sqrt(float(self.m(level)))

    @property
    def factor_scalars(self) -> int:
        """N (2 (c-1) r L + b): the exact O(rN log N) storage."""
        return self.N * (2 * self.W * self.L + self.dcols)

    @property
    def factor_bytes(self) -> int:
        return 8 * self.factor_scalars


# BASELINE.json configs[0..4]
CONFIGS = {
    "c1": HConfig("c1", d=2, L=3, b=64, r=8, nrhs=1, seed=SEED_BASE + 1),
    "c2": HConfig("c2", d=2, L=7, b=64, r=16, nrhs=1, seed=SEED_BASE + 2),
    "c3": HConfig("c3", d=3, L=5, b=64, r=32, nrhs=1, seed=SEED_BASE + 3),
    "c4": HConfig("c4", d=2, L=9, b=64, r=16, nrhs=1, seed=SEED_BASE + 4),
    "c5": HConfig("c5", d=3, L=5, b=64, r=32, nrhs=64, seed=SEED_BASE + 5),
}
# Not a BASELINE config: the standard-admissibility path at C2's
# size (2D, N = 2^20, L = 7, b = 64, r = 16; 27 interaction slots, 9 near-field
# blocks per row) -- the paper's "Standard" columns use the same 1024^2 domain.
EXTRA_CONFIGS = {
    "s2": HConfig("s2", d=2, L=7, b=64, r=16, nrhs=1, seed=SEED_BASE + 12, adm=1),
    # c2 under the paper-strict reading of Def 2.4 (the leaf-parent
    # diagonal blocks, 4 x 64 = 256 square, are dense; low-rank blocks at levels
    # 1..6): exactly the weak structure of depth 6 with leaf 256
    "c2strict": HConfig("c2strict", d=2, L=6, b=256, r=16, nrhs=1, seed=SEED_BASE + 13),
    # the mid-rhs regime (2-16 rhs against the memory floor): the c2 / c4
    # operators with 2, 4, 8 and 16 right-hand sides, and s2 with 16 (the standard
    # structure's tensor-core passes)
    "c2r2": HConfig("c2r2", d=2, L=7, b=64, r=16, nrhs=2, seed=SEED_BASE + 2),
    "c4r2": HConfig("c4r2", d=2, L=9, b=64, r=16, nrhs=2, seed=SEED_BASE + 4),
    "c2r4": HConfig("c2r4", d=2, L=7, b=64, r=16, nrhs=4, seed=SEED_BASE + 2),
    "c2r8": HConfig("c2r8", d=2, L=7, b=64, r=16, nrhs=8, seed=SEED_BASE + 2),
    "c2r16": HConfig("c2r16", d=2, L=7, b=64, r=16, nrhs=16, seed=SEED_BASE + 2),
    "c4r4": HConfig("c4r4", d=2, L=9, b=64, r=16, nrhs=4, seed=SEED_BASE + 4),
    "c4r8": HConfig("c4r8", d=2, L=9, b=64, r=16, nrhs=8, seed=SEED_BASE + 4),
    "c4r16": HConfig("c4r16", d=2, L=9, b=64, r=16, nrhs=16, seed=SEED_BASE + 4),
    "s2r16": HConfig("s2r16", d=2, L=7, b=64, r=16, nrhs=16, seed=SEED_BASE + 12, adm=1),
}

_lib = None
_dev = None


def _load():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libhgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.hgen_value.restype = ctypes.c_double
        lib.hgen_value.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                   ctypes.c_uint64, ctypes.c_double]
        lib.hgen_fill_rowmajor.restype = None
        lib.hgen_fill_rowmajor.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                           ctypes.c_void_p, ctypes.c_int64]
        lib.hgen_fill_x.restype = None
        lib.hgen_fill_x.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64]
        lib.hgen_log_host.restype = ctypes.c_double
        lib.hgen_log_host.argtypes = [ctypes.c_double]
        lib.hgen_cos2pi_host.restype = ctypes.c_double
        lib.hgen_cos2pi_host.argtypes = [ctypes.c_double]
        _lib = lib
    return _lib


def _load_dev():
    global _dev
    if _dev is None:
        path = os.path.join(_HERE, "libhgen_dev.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make`")
        lib = ctypes.CDLL(path)
        lib.hgen_dev_fill_rowmajor.restype = ctypes.c_int
        lib.hgen_dev_fill_rowmajor.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                               ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                               ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        lib.hgen_dev_fill_cols.restype = ctypes.c_int
        lib.hgen_dev_fill_cols.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
                                           ctypes.c_void_p]
        lib.hgen_dev_fill_x.restype = ctypes.c_int
        lib.hgen_dev_fill_x.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p]
        _dev = lib
    return _dev


def value(seed: int, tag: int, level: int, vec: int, idx: int, scale: float = 1.0) -> float:
    return _load().hgen_value(seed, tag, level, vec, idx, scale)


def hgen_log(u: float) -> float:
    return _load().hgen_log_host(u)


def hgen_cos2pi(u: float) -> float:
    return _load().hgen_cos2pi_host(u)


def _ptr(a: np.ndarray) -> int:
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data


def panel(cfg: HConfig, tag: int, level: int, row_begin: int = 0, row_end: int | None = None) -> np.ndarray:
    """Rows [row_begin, row_end) of U_level (TAG_U), V_level (TAG_V) or D (TAG_D)."""
    row_end = cfg.N if row_end is None else row_end
    ncols = cfg.dcols if tag == TAG_D else cfg.W
    scale = 0.125 if tag == TAG_D else cfg.lowrank_scale(level)
    lvl = 0 if tag == TAG_D else level
    out = np.empty((row_end - row_begin, ncols), dtype=np.float64)
    if out.size:
        _load().hgen_fill_rowmajor(cfg.seed, tag, lvl, 0, row_begin, row_end, ncols, scale, _ptr(out), ncols)
    return out


def xblock(cfg: HConfig, nrhs: int | None = None, vec: int = 0, row_begin: int = 0,
           row_end: int | None = None) -> np.ndarray:
    """Rows [row_begin,row_end) of the N x nrhs U(-1,1) block of timing vector `vec`,
    returned as a column-major (Fortran-order) array of shape (rows, nrhs)."""
    nrhs = cfg.nrhs if nrhs is None else nrhs
    row_end = cfg.N if row_end is None else row_end
    rows = row_end - row_begin
    out = np.empty((nrhs, rows), dtype=np.float64)  # C-order (nrhs, rows) == F-order (rows, nrhs)
    if out.size:
        _load().hgen_fill_x(cfg.seed, vec, cfg.N, row_begin, row_end, nrhs, _ptr(out), rows)
    return out.T


def inputs(cfg: HConfig, row_begin: int = 0, row_end: int | None = None):
    """(U[1..L], V[1..L], D) canonical host panels, rows [row_begin,row_end)."""
    U = [panel(cfg, TAG_U, l, row_begin, row_end) for l in range(1, cfg.L + 1)]
    V = [panel(cfg, TAG_V, l, row_begin, row_end) for l in range(1, cfg.L + 1)]
    D = panel(cfg, TAG_D, 0, row_begin, row_end)
    return U, V, D


def dev_fill_panel(cfg: HConfig, tag: int, level: int, row_begin: int, row_end: int,
                   out_ptr: int, ld: int, stream: int = 0) -> None:
    """Device twin of panel(): writes rows [row_begin,row_end) to device memory
    at out_ptr with leading dimension ld (doubles)."""
    ncols = cfg.dcols if tag == TAG_D else cfg.W
    scale = 0.125 if tag == TAG_D else cfg.lowrank_scale(level)
    lvl = 0 if tag == TAG_D else level
    rc = _load_dev().hgen_dev_fill_rowmajor(cfg.seed, tag, lvl, 0, row_begin, row_end, ncols, scale,
                                            out_ptr, ld, stream)
    if rc != 0:
        raise RuntimeError(f"hgen_dev_fill_rowmajor: cuda error {rc}")


def dev_fill_x(cfg: HConfig, nrhs: int, vec: int, row_begin: int, row_end: int, out_ptr: int,
               ld: int, stream: int = 0) -> None:
    rc = _load_dev().hgen_dev_fill_x(cfg.seed, vec, cfg.N, row_begin, row_end, nrhs, out_ptr, ld, stream)
    if rc != 0:
        raise RuntimeError(f"hgen_dev_fill_x: cuda error {rc}")


def dev_fill_operator(cfg: HConfig, panel_fn, row_begin: int, row_end: int, stream: int = 0) -> None:
    """Fill an operator's device panels in place with the synthetic inputs of
    rows [row_begin, row_end).  panel_fn(kind, level) -> (ptr, rows, cols, ld)
    for kind 0 = U_level, 1 = V_level, 2 = D (e.g. paper_2008_12441_b200.hmat.hmat_panel)."""
    for level in range(1, cfg.L + 1):
        for kind, tag in ((0, TAG_U), (1, TAG_V)):
            ptr, rows, cols, ld = panel_fn(kind, level)
            assert rows == row_end - row_begin and cols == cfg.W
            dev_fill_panel(cfg, tag, level, row_begin, row_end, ptr, ld, stream)
    nd = cfg.dcols // cfg.b  # 1 (leaf diagonal) or 3^d near-field panels (standard)
    for e in range(nd):
        ptr, rows, cols, ld = panel_fn(2, e)
        assert rows == row_end - row_begin and cols == cfg.b
        rc = _load_dev().hgen_dev_fill_cols(cfg.seed, TAG_D, 0, 0, row_begin, row_end, cfg.dcols, e * cfg.b,
                                            cfg.b, 0.125, ptr, ld, stream)
        if rc != 0:
            raise RuntimeError(f"hgen_dev_fill_cols: cuda error {rc}")
