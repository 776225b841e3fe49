"""The P > 1 data path on one GPU, rank after rank.

P shards (hmat_dist_t.nranks = P, external_exchange = 1), each built from ITS
rows of the panels, run the split-phase API: hmat_project for every rank, the
exchange buffers summed over ranks here (what ncclAllReduce does inside
hmat_matvec), then hmat_expand for every rank.  No kernel waits on another
rank's kernel (the ranks run one after the other), so this is safe on one GPU
and exercises every multi-GPU code path of the kernels: exchanged levels in
the packed buffer, nodes split across shards, per-shard target bases.  The
library's NCCL layer (dlopen, communicator, in-place fp64 sum on a stream) runs
at one rank in test_nccl_layer_one_rank; a P > 1 NCCL sum needs P GPUs
(tests/test_multigpu_cpu.py covers the layout with real multi-process gloo
communication).
"""
import numpy as np
import pytest

from gen import hgen
from gen.hgen import HConfig
from oracle import oracle
from tests.helpers import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2008_12441_b200 import hmat as hm


@pytest.fixture(autouse=True)
def _wide_passes(monkeypatch):
    """split-phase calls take one pass of right-hand sides: allow the 8-wide
    SIMT kernels (HMAT_MAX_NR=8) so the 5- and 8-rhs cases keep covering them."""
    monkeypatch.setenv("HMAT_MAX_NR", "8")


def sharded_matvec(cfg, P, nrhs):
    hs, xs = [], []
    for g in range(P):
        r0, r1 = g * cfg.N // P, (g + 1) * cfg.N // P
        U, V, D = hgen.inputs(cfg, r0, r1)
        d = hm._dist(nranks=P, rank=g, device=0, external_exchange=True)
        hs.append(hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D, d))
        x = hgen.xblock(cfg, nrhs=nrhs, row_begin=r0, row_end=r1)
        xs.append(torch.from_numpy(np.ascontiguousarray(x.T)).cuda())  # (nrhs, n) = column-major (n, nrhs)
    try:
        cnt = hm.hmat_exchange_size(hs[0], nrhs)
        assert all(hm.hmat_exchange_size(h, nrhs) == cnt for h in hs)
        ex = [torch.zeros(max(cnt, 1), dtype=torch.float64, device="cuda") for _ in range(P)]
        for g in range(P):                       # Step 1 + on-chip Step 2 on every rank
            hm.hmat_project(hs[g], xs[g].t(), ex[g], nrhs)
        torch.cuda.synchronize()
        total = torch.stack(ex).sum(dim=0)       # Steps 2-4 across ranks
        ys = []
        for g in range(P):                       # Step 5 on every rank
            y = torch.empty_like(xs[g])
            hm.hmat_expand(hs[g], xs[g].t(), total, y.t(), nrhs)
            ys.append(y)
        torch.cuda.synchronize()
        return torch.cat(ys, dim=1).t().cpu().numpy(), cnt
    finally:
        for h in hs:
            hm.hmat_destroy(h)


CASES = [
    (HConfig("p2d", d=2, L=4, b=16, r=4, seed=301), 2, 1),
    (HConfig("p2d", d=2, L=4, b=16, r=4, seed=301), 4, 3),
    (HConfig("p2d", d=2, L=4, b=16, r=4, seed=301), 8, 2),
    (HConfig("p2d", d=2, L=4, b=16, r=4, seed=301), 16, 1),
    (HConfig("p3d", d=3, L=3, b=8, r=3, seed=302), 8, 1),
    (HConfig("p3d", d=3, L=3, b=8, r=3, seed=302), 2, 5),
    (HConfig("p1d", d=1, L=7, b=4, r=2, seed=303), 8, 2),
    (HConfig("podd", d=2, L=3, b=7, r=3, seed=304), 4, 1),
    (HConfig("pdmma", d=3, L=3, b=64, r=32, seed=305), 8, 64),   # tensor-core path
    (HConfig("pdmma2", d=2, L=4, b=64, r=32, seed=306), 4, 20),  # tensor-core path, ragged rhs
    (HConfig("pdmma3", d=2, L=4, b=64, r=16, seed=309), 8, 64),  # tensor-core path, W = 48
    (HConfig("pdmma3", d=2, L=4, b=64, r=16, seed=309), 4, 7),   # 16-wide pass, W = 48
    (HConfig("pdmma", d=3, L=3, b=64, r=32, seed=305), 2, 12),   # 16-wide pass, W = 224
    (HConfig("pdmma", d=3, L=3, b=64, r=32, seed=305), 8, 8),    # 8-wide pass, W = 224
    (HConfig("pdmma3", d=2, L=4, b=64, r=16, seed=309), 8, 6),   # 8-wide pass, W = 48
]


@pytest.mark.parametrize("cfg,P,nrhs", CASES, ids=lambda v: getattr(v, "name", str(v)))
def test_sharded_split_phase_matches_oracle(cfg, P, nrhs):
    y, cnt = sharded_matvec(cfg, P, nrhs)
    U, V, D = hgen.inputs(cfg)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, hgen.xblock(cfg, nrhs=nrhs))
    assert_parity(y, ref)
    assert cnt > 0


def test_sharded_equals_single_gpu_c2_shape():
    """P = 4 shards of a C2-sized operator agree with the P = 1 operator."""
    cfg = HConfig("c2s", d=2, L=6, b=64, r=16, seed=307)
    y4, _ = sharded_matvec(cfg, 4, 1)
    U, V, D = hgen.inputs(cfg)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        x = torch.from_numpy(np.ascontiguousarray(hgen.xblock(cfg, nrhs=1)[:, 0])).cuda()
        y1 = torch.empty_like(x)
        hm.hmat_matvec(h, x, y1)
        assert_parity(y4[:, 0], y1.cpu().numpy())
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("count", [1, 4097, 1 << 20])
def test_nccl_layer_one_rank(count):
    torch.zeros(1, device="cuda")                     # torch's NCCL / context first, as bench.py
    hm.hmat_nccl_selftest(0, count)


def test_external_exchange_requires_split_api():
    cfg = HConfig("p", d=2, L=2, b=4, r=2, seed=308)
    U, V, D = hgen.inputs(cfg, 0, cfg.N // 2)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D, hm._dist(nranks=2, rank=0, device=0, external_exchange=True))
    try:
        x = torch.zeros(cfg.N // 2, dtype=torch.float64, device="cuda")
        with pytest.raises(hm.HMatError) as ei:
            hm.hmat_matvec(h, x, torch.empty_like(x))
        assert ei.value.status == hm.HMAT_ERR_UNSUPPORTED
    finally:
        hm.hmat_destroy(h)


def peer_split_matvec(cfg, P, nrhs, reps=2):
    """HMAT_EXCHANGE_PEER on one GPU: every rank's project kernel pushes its
    exchange levels into all mailboxes and raises its flags; then every rank's
    expand kernel consumes them (projects of all ranks first, so no kernel ever
    waits for another one on this single GPU)."""
    hs, xs = [], []
    for g in range(P):
        r0, r1 = g * cfg.N // P, (g + 1) * cfg.N // P
        U, V, D = hgen.inputs(cfg, r0, r1)
        d = hm._dist(nranks=P, rank=g, device=0, exchange=hm.HMAT_EXCHANGE_PEER)
        hs.append(hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D, d))
        xs.append(torch.from_numpy(np.ascontiguousarray(hgen.xblock(cfg, nrhs=nrhs, row_begin=r0,
                                                                    row_end=r1).T)).cuda())
    try:
        for h in hs:
            hm.hmat_peer_connect_local(h, hs)
        out = []
        for rep in range(reps):  # several passes: mailbox parities alternate
            for g in range(P):
                hm.hmat_project(hs[g], xs[g].t(), None, nrhs)
            ys = []
            for g in range(P):
                y = torch.empty_like(xs[g])
                hm.hmat_expand(hs[g], xs[g].t(), None, y.t(), nrhs)
                ys.append(y)
            torch.cuda.synchronize()
            out.append(torch.cat(ys, dim=1).t().cpu().numpy())
        return out
    finally:
        for h in hs:
            hm.hmat_destroy(h)


@pytest.mark.parametrize("cfg,P,nrhs", [
    (HConfig("q2d", d=2, L=4, b=16, r=4, seed=401), 2, 1),
    (HConfig("q2d", d=2, L=4, b=16, r=4, seed=401), 8, 3),
    (HConfig("q3d", d=3, L=3, b=8, r=3, seed=402), 4, 2),
    (HConfig("q3d", d=3, L=3, b=64, r=32, seed=403), 8, 1),
    (HConfig("q1d", d=1, L=7, b=4, r=2, seed=404), 16, 8),
    # tensor-core path: the project's last CTA pushes, a rank-ordered sum kernel precedes expand
    (HConfig("q3d", d=3, L=3, b=64, r=32, seed=403), 2, 64),
    (HConfig("q3d", d=3, L=3, b=64, r=32, seed=403), 8, 20),     # 32-wide pass
    (HConfig("qw48", d=2, L=4, b=64, r=16, seed=405), 4, 7),     # W = 48, 16-wide pass
], ids=lambda v: getattr(v, "name", str(v)))
def test_peer_exchange_matches_oracle(cfg, P, nrhs):
    outs = peer_split_matvec(cfg, P, nrhs)
    U, V, D = hgen.inputs(cfg)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, hgen.xblock(cfg, nrhs=nrhs))
    for y in outs:
        assert_parity(y, ref)
    assert np.array_equal(outs[0], outs[1])  # deterministic (rank-order sums)


def test_peer_exchange_needs_connection():
    cfg = HConfig("qc", d=2, L=2, b=4, r=2, seed=405)
    U, V, D = hgen.inputs(cfg, 0, cfg.N // 2)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D,
                       hm._dist(nranks=2, rank=0, device=0, exchange=hm.HMAT_EXCHANGE_PEER))
    try:
        x = torch.zeros(cfg.N // 2, dtype=torch.float64, device="cuda")
        with pytest.raises(hm.HMatError) as ei:
            hm.hmat_project(h, x, None)
        assert ei.value.status == hm.HMAT_ERR_INVALID
        assert len(hm.hmat_peer_export(h)) == 64
    finally:
        hm.hmat_destroy(h)


# ---- standard admissibility with P > 1 -------------------------------
# Cross-rank interaction pairs exist at every level along the slice boundaries and
# the near field of a boundary leaf reaches other ranks' x: both travel in the
# packed buffer of csrc/std_exchange.h (summed over ranks here).

def sharded_std_matvec(cfg, P, nrhs):
    hs, xs = [], []
    for g in range(P):
        r0, r1 = g * cfg.N // P, (g + 1) * cfg.N // P
        U, V, Dn = hgen.inputs(cfg, r0, r1)
        d = hm._dist(nranks=P, rank=g, device=0, external_exchange=True)
        hs.append(hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, U, V, Dn, d))
        x = hgen.xblock(cfg, nrhs=nrhs, row_begin=r0, row_end=r1)
        xs.append(torch.from_numpy(np.ascontiguousarray(x.T)).cuda())
    try:
        cnt = hm.hmat_exchange_size(hs[0], nrhs)
        assert all(hm.hmat_exchange_size(h, nrhs) == cnt for h in hs)
        ex = [torch.zeros(max(cnt, 1), dtype=torch.float64, device="cuda") for _ in range(P)]
        for g in range(P):
            hm.hmat_project(hs[g], xs[g].t(), ex[g], nrhs)
        torch.cuda.synchronize()
        total = torch.stack(ex).sum(dim=0)
        ys = []
        for rep in range(2):  # twice: the buffers are re-zeroed / re-packed per pass
            ys = []
            for g in range(P):
                y = torch.full_like(xs[g], float("nan"))
                hm.hmat_expand(hs[g], xs[g].t(), total, y.t(), nrhs)
                ys.append(y)
        torch.cuda.synchronize()
        return torch.cat(ys, dim=1).t().cpu().numpy(), cnt
    finally:
        for h in hs:
            hm.hmat_destroy(h)


STD_CASES = [
    (HConfig("s2d", d=2, L=4, b=8, r=3, adm=1, seed=311), 2, 1),
    (HConfig("s2d", d=2, L=4, b=8, r=3, adm=1, seed=311), 4, 2),
    (HConfig("s2d", d=2, L=4, b=8, r=3, adm=1, seed=311), 8, 1),
    (HConfig("s2d", d=2, L=4, b=8, r=3, adm=1, seed=311), 16, 3),
    (HConfig("s1d", d=1, L=6, b=4, r=2, adm=1, seed=312), 8, 1),    # 1D: nodes spanning ranks at levels 2, 3
    (HConfig("s1d", d=1, L=6, b=4, r=2, adm=1, seed=312), 32, 2),
    (HConfig("s3d", d=3, L=3, b=4, r=1, adm=1, seed=313), 8, 1),
    (HConfig("s3d", d=3, L=3, b=4, r=1, adm=1, seed=313), 64, 1),   # one level-2 node per rank
    (HConfig("sodd", d=2, L=3, b=7, r=2, adm=1, seed=314), 4, 1),   # odd leaf: halo x parity
    (HConfig("s64", d=2, L=5, b=64, r=8, adm=1, seed=315), 8, 1),
]


# the tensor-core path (from 5 rhs; W = 27 r = 432 in 2-D, 3 r = 48 in 1-D):
# cross-rank z entries scattered by the DMMA project into the packed buffer,
# remote neighbours' x read by tensor TMA from its halo region, the received
# entries unpacked into the fragment-major Zt (kernels_dmma.cu)
STD_DMMA_CASES = [
    (HConfig("sdm2", d=2, L=4, b=64, r=16, adm=1, seed=316), 2, 5),    # 8-wide pass
    (HConfig("sdm2", d=2, L=4, b=64, r=16, adm=1, seed=316), 4, 12),   # 16-wide
    (HConfig("sdm2", d=2, L=4, b=64, r=16, adm=1, seed=316), 8, 20),   # 32-wide
    (HConfig("sdm2", d=2, L=4, b=64, r=16, adm=1, seed=316), 16, 64),  # one level-2 node per rank
    (HConfig("sdm1", d=1, L=6, b=64, r=16, adm=1, seed=317), 8, 9),    # 1D: nodes spanning ranks
]


@pytest.mark.parametrize("cfg,P,nrhs", STD_CASES + STD_DMMA_CASES, ids=lambda v: getattr(v, "name", str(v)))
def test_standard_sharded_split_phase_matches_oracle(cfg, P, nrhs):
    y, cnt = sharded_std_matvec(cfg, P, nrhs)
    U, V, Dn = hgen.inputs(cfg)
    ref = oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, hgen.xblock(cfg, nrhs=nrhs))
    assert_parity(y, ref)
    assert cnt > 0


def sharded_std_gemv_t(cfg, P, nrhs, alpha, beta, y0):
    """H^T with P shards, rank after rank through the split-phase op calls: the
    buffer carries the z entries and the products (D_{S,T})^T x_S of the cross
    near-field pairs; hmat_expand_op adds the incoming ones."""
    hs, xs, ys = [], [], []
    for g in range(P):
        r0, r1 = g * cfg.N // P, (g + 1) * cfg.N // P
        U, V, Dn = hgen.inputs(cfg, r0, r1)
        d = hm._dist(nranks=P, rank=g, device=0, external_exchange=True)
        hs.append(hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, U, V, Dn, d))
        x = hgen.xblock(cfg, nrhs=nrhs, row_begin=r0, row_end=r1)
        xs.append(torch.from_numpy(np.ascontiguousarray(x.T)).cuda())
        ys.append(torch.from_numpy(np.ascontiguousarray(y0[r0:r1].T)).cuda())
    try:
        cnt = hm.hmat_exchange_size_op(hs[0], 1, nrhs)
        assert all(hm.hmat_exchange_size_op(h, 1, nrhs) == cnt for h in hs)
        ex = [torch.zeros(max(cnt, 1), dtype=torch.float64, device="cuda") for _ in range(P)]
        for g in range(P):
            hm.hmat_project_op(hs[g], 1, xs[g].t(), ex[g], nrhs)
        torch.cuda.synchronize()
        total = torch.stack(ex).sum(dim=0)
        for g in range(P):
            hm.hmat_expand_op(hs[g], 1, alpha, xs[g].t(), total, beta, ys[g].t(), nrhs)
        torch.cuda.synchronize()
        return torch.cat(ys, dim=1).t().cpu().numpy(), cnt
    finally:
        for h in hs:
            hm.hmat_destroy(h)


@pytest.mark.parametrize("cfg,P,nrhs", [STD_CASES[0], STD_CASES[1], STD_CASES[3], STD_CASES[4], STD_CASES[5],
                                        STD_CASES[6], STD_CASES[8], STD_CASES[9]] + STD_DMMA_CASES,
                         ids=lambda v: getattr(v, "name", str(v)))
def test_standard_sharded_transpose_matches_oracle(cfg, P, nrhs):
    """Standard admissibility, H^T with P > 1 (PAPER.md:961-969 GEMV "T"): the
    shards' y = alpha H^T x + beta y0 vs the transposed oracle block loop."""
    rng = np.random.default_rng(7)
    y0 = rng.standard_normal((cfg.N, nrhs))
    y, cnt = sharded_std_gemv_t(cfg, P, nrhs, 0.75, -0.5, y0)
    U, V, Dn = hgen.inputs(cfg)
    ref = 0.75 * oracle.std_matvec_t(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, hgen.xblock(cfg, nrhs=nrhs)) - 0.5 * y0
    assert_parity(y, ref)
    assert cnt > 0


# ---- failure behaviour of the PEER exchange ------------------------------------------

def _peer_pair(cfg, monkeypatch, timeout_ms):
    monkeypatch.setenv("HMAT_PEER_TIMEOUT_MS", str(timeout_ms))
    P = 2
    hs, xs = [], []
    for g in range(P):
        r0, r1 = g * cfg.N // P, (g + 1) * cfg.N // P
        U, V, D = hgen.inputs(cfg, r0, r1)
        hs.append(hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D,
                                 hm._dist(nranks=P, rank=g, device=0, exchange=hm.HMAT_EXCHANGE_PEER)))
        xs.append((r0, r1))
    for h in hs:
        hm.hmat_peer_connect_local(h, hs)
    return hs, xs


@pytest.mark.parametrize("cfg,nrhs", [(HConfig("t2d", d=2, L=3, b=16, r=4, seed=421), 1),        # SIMT expand waits
                                      (HConfig("t3d", d=3, L=2, b=64, r=32, seed=422), 64)],     # tensor-core peer_sum waits
                         ids=["simt", "dmma"])
def test_peer_flag_timeout_is_an_error_not_a_fault(cfg, nrhs, monkeypatch):
    """A rank whose peer never raises its flag: the bounded wait gives up after
    HMAT_PEER_TIMEOUT_MS, the handle reports HMAT_ERR_NCCL (naming the missing
    rank) at hmat_synchronize, once, and the CUDA context stays usable (no trap):
    later work on the device, including another H-matvec, is correct."""
    hs, rows = _peer_pair(cfg, monkeypatch, 300)
    try:
        r0, r1 = rows[0]
        x = torch.from_numpy(np.ascontiguousarray(hgen.xblock(cfg, nrhs=nrhs, row_begin=r0, row_end=r1).T)).cuda()
        y = torch.empty_like(x)
        hm.hmat_project(hs[0], x.t(), None, nrhs)          # rank 0 pushes and raises its flags
        hm.hmat_expand(hs[0], x.t(), None, y.t(), nrhs)    # ... and waits for rank 1's, which never come
        with pytest.raises(hm.HMatError) as ei:
            hm.hmat_synchronize(hs[0])
        assert ei.value.status == hm.HMAT_ERR_NCCL
        assert "rank 1" in str(ei.value) and "not raised" in str(ei.value)
        hm.hmat_synchronize(hs[0])                          # reported once
        assert torch.isfinite(y).all()
    finally:
        for h in hs:
            hm.hmat_destroy(h)
    assert float(torch.ones(1000, device="cuda", dtype=torch.float64).sum()) == 1000.0
    c = HConfig("after", d=2, L=3, b=16, r=4, seed=423)
    U, V, D = hgen.inputs(c)
    x = hgen.xblock(c, nrhs=1)[:, 0]
    h = hm.hmat_create(c.L, c.d, c.b, c.r, U, V, D)
    try:
        xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
        yd = torch.empty_like(xd)
        hm.hmat_matvec(h, xd, yd)
        assert_parity(yd.cpu().numpy(), oracle.matvec(c.d, c.L, c.b, c.r, U, V, D, x))
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("cfg,nrhs", [(HConfig("m2d", d=2, L=3, b=16, r=4, seed=424), 2),
                                      (HConfig("m3d", d=3, L=2, b=64, r=32, seed=425), 8)],
                         ids=["simt", "dmma"])
def test_peer_dense_only_parts_do_not_wait(cfg, nrhs, monkeypatch):
    """hmat_matvec_parts(mask = 0, dense = 1) on a PEER handle runs no project,
    so no rank raises a flag: nothing may wait for one (the tensor-core path
    skips its mailbox sum).  Rank 0 alone gets y = D x of its rows, no error."""
    hs, rows = _peer_pair(cfg, monkeypatch, 2000)
    try:
        r0, r1 = rows[0]
        xh = hgen.xblock(cfg, nrhs=nrhs)
        x = torch.from_numpy(np.ascontiguousarray(xh[r0:r1].T)).cuda()
        y = torch.empty_like(x)
        hm.hmat_matvec_parts(hs[0], x.t(), y.t(), 0, True, nrhs)
        hm.hmat_synchronize(hs[0])
        U, V, D = hgen.inputs(cfg)
        ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, xh, level_mask=0, dense=True)
        assert_parity(y.t().cpu().numpy(), ref[r0:r1])
    finally:
        for h in hs:
            hm.hmat_destroy(h)


def test_comm_info_without_nccl():
    cfg = HConfig("ci", d=2, L=2, b=4, r=2, seed=426)
    U, V, D = hgen.inputs(cfg, cfg.N // 4, cfg.N // 2)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D, hm._dist(nranks=4, rank=1, device=0,
                                                                       external_exchange=True))
    try:
        assert hm.hmat_comm_info(h) == (4, 1)
    finally:
        hm.hmat_destroy(h)
