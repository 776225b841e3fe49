"""BASELINE configs at FULL size, compared in full (every row, every column).

The oracle side is `oracle.matvec_generated`: the block loop of eq:hmat-vec-add
 with every factor entry generated on demand from the seeded
recipe (gen/hgen.h) on all host cores -- bit-identical to `oracle.matvec` on the
generated panels (tests/test_oracle_pins.py::test_matvec_generated_*), so it
carries all of the block loop's pins, and it needs no factor memory on the host.
Each oracle y is computed once per session and reused by the P = 1 and the
sharded checks of the same config.

GPU side, in the bench's launch configuration (device-generated panels, default
plan):
  * P = 1: c3, c4 (BASELINE configs[2], [3]; single vector) and c5 (configs[4],
    64 right-hand sides on the FP64 tensor-core path), and the bench's c2strict
    line (c2 under the paper-strict Def 2.4: the weak structure of depth 6 with
    256-point leaves, dense blocks streamed in 64-column chunks), through
    hmat_matvec.  A
    full comparison covers every expand item, both sides of every project
    CTA-range boundary, every node split across CTAs, and the first and last
    leaves.
  * P = 8 shards, rank after rank on this one GPU through the split-phase API
    (hmat_project -> the exchange buffers summed over ranks -> hmat_expand):
    c4 with two level-2 nodes per shard (the paper's 2D example)
    and c3 with one level-1 octant per shard (BASELINE configs[2]).  The 8 shards
    hold exactly the P = 1 operator's 124.55 / 38.65 GB.
Tolerance: the north star's relative l2 <= 1e-12 per column, and every element
within 1e-12 * max|y_ref| of its column (tests/helpers.assert_parity).
"""
import time

import numpy as np
import pytest

from gen import hgen
from gen.hgen import CONFIGS
from oracle import oracle
from tests.helpers import assert_parity, device_operator

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2008_12441_b200 import hmat as hm

CFGS = {**CONFIGS, "c2strict": hgen.EXTRA_CONFIGS["c2strict"]}
XVEC = {"c2": 3, "c3": 3, "c4": 3, "c5": 0, "c2strict": 3}  # timing-vector index of the x under test
_REF = {}


def oracle_y(name):
    """Full oracle y of config `name` for its test vector (host, all cores)."""
    if name not in _REF:
        cfg = CFGS[name]
        x = hgen.xblock(cfg, nrhs=cfg.nrhs, vec=XVEC[name])
        t0 = time.perf_counter()
        y = oracle.matvec_generated(cfg, x)
        print(f"[oracle] {name}: full y in {time.perf_counter() - t0:.1f} s on {oracle.host_threads()} threads")
        _REF[name] = (np.asfortranarray(x), y if y.ndim == 2 else y[:, None])
    return _REF[name]


def need(bytes_):
    free, _ = torch.cuda.mem_get_info()
    if free < bytes_:
        pytest.skip(f"needs {bytes_ / 1e9:.0f} GB of device memory")


@pytest.mark.parametrize("name", ["c2strict", "c3", "c4", "c5"])
def test_full_size_in_full(name):
    cfg = CFGS[name]
    need(cfg.factor_bytes * 1.05 + 4 * 8 * cfg.N * cfg.nrhs)
    x, ref = oracle_y(name)
    h = device_operator(cfg, hm)
    try:
        X = torch.empty(cfg.nrhs, cfg.N, dtype=torch.float64, device="cuda")   # column-major N x nrhs
        hgen.dev_fill_x(cfg, cfg.nrhs, XVEC[name], 0, cfg.N, X.data_ptr(), cfg.N)
        Y = torch.empty_like(X)
        hm.hmat_matvec(h, X.t(), Y.t(), cfg.nrhs)
        torch.cuda.synchronize()
        assert np.array_equal(X.t().cpu().numpy(), x)   # the same x on both sides
        assert hm.hmat_launches_per_matvec(h, cfg.nrhs) == 2
        assert_parity(Y.t().cpu().numpy(), ref)
    finally:
        hm.hmat_destroy(h)
        torch.cuda.empty_cache()


@pytest.mark.parametrize("name,P", [("c4", 8), ("c3", 8), ("c2", 8), ("c4", 2)])
def test_sharded_full_size_in_full(name, P):
    """P shards of a full-size BASELINE operator, every rank's rows compared."""
    cfg = CFGS[name]
    need(cfg.factor_bytes * 1.05 + 6 * 8 * cfg.N)
    x, ref = oracle_y(name)
    hs, xs = [], []
    try:
        for g in range(P):
            d = hm._dist(nranks=P, rank=g, device=0, external_exchange=True)
            h = device_operator(cfg, hm, d)
            hs.append(h)
            r0, r1 = hm.hmat_local_rows(h)
            assert (r0, r1) == (g * cfg.N // P, (g + 1) * cfg.N // P)   # block-row rule
            xv = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
            hgen.dev_fill_x(cfg, 1, XVEC[name], r0, r1, xv.data_ptr(), r1 - r0)
            xs.append(xv)
        cnt = hm.hmat_exchange_size(hs[0], 1)
        # exchanged levels: those whose parent spans ranks (c^(l-1) < P), target-major
        cross = [lvl for lvl in range(1, cfg.L + 1) if cfg.c ** (lvl - 1) < P]
        assert cnt == sum(cfg.c ** lvl for lvl in cross) * hm.hmat_plan_query(cfg.L, cfg.d, cfg.b, cfg.r, P, 0).W_pitch
        ex = [torch.zeros(cnt, dtype=torch.float64, device="cuda") for _ in range(P)]
        for g in range(P):                       # Step 1 + on-chip Step 2 on every rank
            hm.hmat_project(hs[g], xs[g], ex[g], 1)
        torch.cuda.synchronize()
        total = ex[0].clone()                    # Steps 2-4 across ranks (rank order)
        for g in range(1, P):
            total += ex[g]
        ys = []
        for g in range(P):                       # Step 5 on every rank
            y = torch.empty_like(xs[g])
            hm.hmat_expand(hs[g], xs[g], total, y, 1)
            ys.append(y)
        torch.cuda.synchronize()
        got = torch.cat(ys).cpu().numpy()
        assert_parity(got, ref[:, 0])
    finally:
        for h in hs:
            hm.hmat_destroy(h)
        torch.cuda.empty_cache()
