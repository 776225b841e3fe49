"""Memory bounds of the kernels, checked with guard zones (compute-sanitizer is
not available on the GPU pool).

x, y and the split-phase exchange buffer are interior slices of larger device
allocations.  The guard zones around x hold NaN: a kernel that lets any value
outside x reach y (an out-of-range row, a padding column multiplied by zero --
NaN * 0 = NaN) fails parity.  The guard zones around y and the exchange buffer
hold a bit pattern that must survive every call bit for bit: a store outside
the caller's buffer fails.  y's interior starts as NaN where beta = 0 (the
result must not read it).  Every kernel variant: SIMT weak (ragged leaves, odd
W, several passes of right-hand sides), standard admissibility (op = H, H^T),
the paper-strict structure, the DMMA path (ragged last pass), split-phase P > 1.
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

G = 4096                        # guard doubles on each side (32 KB; keeps 512-byte alignment)
MARK = np.float64(-1.2345e300)  # y / exchange guard value


def guarded(n, k, guard_value, fill, shift=0):
    """(base, view): a device (n, k) column-major view at offset G + shift of a
    buffer of n k + 2 G + shift doubles (shift = 1: 8-byte aligned only); guards
    (the first G and last G doubles) = guard_value, interior = fill."""
    base = torch.full((n * k + 2 * G + shift,), float(guard_value), dtype=torch.float64, device="cuda")
    v = base[G + shift:G + shift + n * k].view(k, n).t()
    if np.isscalar(fill):
        v.fill_(float(fill))
    else:
        v.copy_(torch.from_numpy(np.asfortranarray(np.asarray(fill).reshape(n, k))))
    return base, v


def guards_intact(base, value):
    g = torch.cat([base[:G], base[-G:]]).cpu().numpy()
    return np.array_equal(g.view(np.int64), np.full(2 * G, value, dtype=np.float64).view(np.int64))


def run_checked(h, n, x, ref, trans=0, alpha=1.0, beta=0.0, y0=None, shift=0):
    k = x.shape[1]
    xb, xv = guarded(n, k, np.nan, x, shift)
    yb, yv = guarded(n, k, MARK, np.nan if y0 is None else y0, shift)
    hm.hmat_gemv(h, trans, alpha, xv, beta, yv)
    torch.cuda.synchronize()
    assert guards_intact(yb, MARK), "a store landed outside y"
    assert torch.isnan(torch.cat([xb[:G], xb[-G:]])).all()  # x guards untouched too
    want = alpha * ref + (0.0 if y0 is None else beta * y0)
    assert_parity(yv.cpu().numpy(), want)


WEAK = [HConfig("w1", d=2, L=3, b=7, r=5, seed=1701),      # odd leaf, odd W = 15
        HConfig("w2", d=3, L=2, b=1, r=7, seed=1702),      # 1-row leaves
        HConfig("w3", d=1, L=6, b=4, r=3, seed=1703),      # W = 3
        HConfig("w4", d=2, L=3, b=64, r=86, seed=1704),    # W = 258 > consumer threads
        HConfig("w5", d=2, L=4, b=64, r=16, seed=1705)]    # the c2 / c4 shape (W = 48)


@pytest.mark.parametrize("cfg", WEAK, ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [1, 3, 9])
@pytest.mark.parametrize("shift", [0, 1])  # 1: x / y only 8-byte aligned (staged internally)
def test_weak_guards(cfg, nrhs, shift):
    U, V, D = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        run_checked(h, cfg.N, x, oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x), shift=shift)
        y0 = np.random.default_rng(3).standard_normal(x.shape)
        run_checked(h, cfg.N, x, oracle.matvec_t(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x), trans=1,
                    alpha=0.5, beta=-2.0, y0=y0, shift=shift)
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("cfg", [HConfig("d2r16", d=2, L=4, b=64, r=16, seed=1711),   # W = 48
                                 HConfig("d3r32", d=3, L=2, b=64, r=32, seed=1712)],  # W = 224
                         ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [16, 70])
def test_dmma_guards(cfg, nrhs):
    U, V, D = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        assert hm.hmat_launches_per_matvec(h, nrhs) == 2 * ((nrhs + 63) // 64)  # the DMMA path
        run_checked(h, cfg.N, x, oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x))
        run_checked(h, cfg.N, x, oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x), shift=1)
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("cfg", [HConfig("s1", d=2, L=3, b=5, r=3, adm=1, seed=1721),
                                 HConfig("s2", d=3, L=2, b=4, r=2, adm=1, seed=1722),
                                 HConfig("s3", d=1, L=5, b=3, r=2, adm=1, seed=1723)], ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [1, 3])
def test_standard_guards(cfg, nrhs):
    U, V, Dn = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, U, V, Dn)
    try:
        run_checked(h, cfg.N, x, oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x))
        run_checked(h, cfg.N, x, oracle.std_matvec_t(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x), trans=1, shift=1)
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("d,L,b,r", [(2, 3, 5, 2), (2, 3, 64, 4)])  # odd leaf; leaf 256 (chunked dense)
def test_strict_guards(d, L, b, r):
    c = 1 << d
    N = b * c ** L
    W = (c - 1) * r
    rng = np.random.default_rng(1730 + b)
    U = [rng.standard_normal((N, W)) / 8 for _ in range(L - 1)]
    V = [rng.standard_normal((N, W)) / 8 for _ in range(L - 1)]
    Dc = rng.standard_normal((N, c * b)) / 8
    x = rng.uniform(-1, 1, (N, 3))
    h = hm.hmat_create_strict(L, d, b, r, U, V, Dc)
    try:
        run_checked(h, N, x, oracle.matvec_strict(d, L, b, r, U, V, Dc, x))
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("cfg,P", [(HConfig("m1", d=2, L=3, b=4, r=2, seed=1741), 4),
                                   (HConfig("m2", d=2, L=3, b=4, r=2, adm=1, seed=1742), 4)],
                         ids=lambda v: getattr(v, "name", str(v)))
def test_split_phase_exchange_guards(cfg, P):
    """P shards rank after rank through hmat_project / hmat_expand: the exchange
    buffer each rank writes is a guarded slice; its guards and y's survive."""
    nrhs = 2
    n = cfg.N // P
    x = hgen.xblock(cfg, nrhs=nrhs)
    U, V, D = hgen.inputs(cfg)
    create = hm.hmat_create_standard if cfg.adm else hm.hmat_create
    hs = []
    try:
        for g in range(P):
            Ug, Vg, Dg = hgen.inputs(cfg, g * n, (g + 1) * n)
            hs.append(create(cfg.L, cfg.d, cfg.b, cfg.r, Ug, Vg, Dg,
                             hm._dist(nranks=P, rank=g, device=0, external_exchange=True)))
        cnt = hm.hmat_exchange_size(hs[0], nrhs)
        assert cnt > 0
        bufs, xs = [], []
        for g in range(P):
            xb, xv = guarded(n, nrhs, np.nan, x[g * n:(g + 1) * n])
            eb = torch.full((cnt + 2 * G,), float(MARK), dtype=torch.float64, device="cuda")
            hm.hmat_project(hs[g], xv, eb[G:G + cnt], nrhs)
            bufs.append(eb)
            xs.append((xb, xv))
        torch.cuda.synchronize()
        for eb in bufs:
            assert guards_intact(eb, MARK), "project stored outside the exchange buffer"
        total = sum(eb[G:G + cnt] for eb in bufs)
        ys = []
        for g in range(P):
            yb, yv = guarded(n, nrhs, MARK, np.nan)
            hm.hmat_expand(hs[g], xs[g][1], total, yv, nrhs)
            ys.append((yb, yv))
        torch.cuda.synchronize()
        for yb, _ in ys:
            assert guards_intact(yb, MARK), "expand stored outside y"
        y = np.concatenate([yv.cpu().numpy() for _, yv in ys])
        ref = (oracle.std_matvec if cfg.adm else oracle.matvec)(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
        assert_parity(y, ref)
    finally:
        for h in hs:
            hm.hmat_destroy(h)
