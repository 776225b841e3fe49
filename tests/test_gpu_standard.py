"""GPU parity of the standard-admissibility path against the
oracle's block loop (tests/test_oracle_std.py pins that oracle)."""
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


def run_std(cfg, nrhs, **parts):
    U, V, Dn = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, U, V, Dn)
    try:
        xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        yd = torch.empty_like(xd)
        if parts:
            hm.hmat_matvec_parts(h, xd.t(), yd.t(), **parts)
        else:
            hm.hmat_matvec(h, xd.t(), yd.t())
        torch.cuda.synchronize()
        return yd.t().cpu().numpy(), (U, V, Dn, x)
    finally:
        hm.hmat_destroy(h)


STD = [HConfig(f"std{d}{L}{b}{r}", d=d, L=L, b=b, r=r, adm=1, seed=700 + 31 * d + 7 * L + b + r)
       for d, L, b, r in [(1, 5, 4, 2), (1, 8, 2, 3), (2, 2, 4, 2), (2, 3, 8, 2), (2, 4, 16, 4), (2, 3, 7, 3),
                          (3, 2, 4, 1), (3, 3, 8, 1), (2, 5, 64, 8)]]


@pytest.mark.parametrize("cfg", STD, ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [1, 3])
def test_standard_admissibility_parity(cfg, nrhs):
    y, (U, V, Dn, x) = run_std(cfg, nrhs)
    ref = oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x)
    assert_parity(y, ref)


def test_standard_near_field_only_and_far_field_only():
    """level parts: the dense near field alone and the far field alone."""
    cfg = HConfig("stdp", d=2, L=4, b=8, r=3, adm=1, seed=777)
    U, V, Dn = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=1)
    Z = [np.zeros_like(u) for u in U]
    y, _ = run_std(cfg, 1, level_mask=0, dense=True)
    assert_parity(y, oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, Z, Z, Dn, x))
    y, _ = run_std(cfg, 1, level_mask=(1 << cfg.L) - 1, dense=False)
    assert_parity(y, oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, np.zeros_like(Dn), x))


def run_std_gemv(cfg, nrhs, trans, alpha, beta, y0=None):
    U, V, Dn = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, U, V, Dn)
    try:
        xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        yd = torch.from_numpy(np.ascontiguousarray(y0.T)).cuda() if y0 is not None else torch.full_like(xd, float("nan"))
        hm.hmat_gemv(h, trans, alpha, xd.t(), beta, yd.t())
        torch.cuda.synchronize()
        return yd.t().cpu().numpy(), (U, V, Dn, x)
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("cfg", STD, ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [1, 3])
def test_standard_transposed_parity(cfg, nrhs):
    """H^T x (GEMV "T") against the oracle's transposed loop;
    beta = 0 must not read the NaN-filled y."""
    y, (U, V, Dn, x) = run_std_gemv(cfg, nrhs, 1, 1.0, 0.0)
    assert_parity(y, oracle.std_matvec_t(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x))


def test_standard_gemv_alpha_beta_both_ops():
    cfg = HConfig("stdab", d=2, L=4, b=8, r=3, adm=1, seed=781)
    y0 = np.random.default_rng(8).standard_normal((cfg.N, 2))
    for trans, fn in ((0, oracle.std_matvec), (1, oracle.std_matvec_t)):
        y, (U, V, Dn, x) = run_std_gemv(cfg, 2, trans, -0.75, 1.5, y0)
        assert_parity(y, -0.75 * fn(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x) + 1.5 * y0)


def test_standard_adjoint_identity_gpu():
    """<y', H x> = <H^T y', x> with both products on the GPU (3D, b = 64)."""
    cfg = HConfig("stdadj", d=3, L=2, b=64, r=2, adm=1, seed=782)
    U, V, Dn = hgen.inputs(cfg)
    h = hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, U, V, Dn)
    try:
        g = torch.Generator(device="cpu").manual_seed(9)
        x = torch.randn(cfg.N, dtype=torch.float64, generator=g).cuda()
        yp = torch.randn(cfg.N, dtype=torch.float64, generator=g).cuda()
        hx, hty = torch.empty_like(x), torch.empty_like(x)
        hm.hmat_gemv(h, 0, 1.0, x, 0.0, hx)
        hm.hmat_gemv(h, 1, 1.0, yp, 0.0, hty)
        torch.cuda.synchronize()
        lhs, rhs = float(yp @ hx), float(hty @ x)
        assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    finally:
        hm.hmat_destroy(h)


def test_standard_unsupported_cases():
    """The in-kernel peer exchange is weak-admissibility only."""
    cfg = HConfig("stdu", d=2, L=3, b=4, r=2, adm=1, seed=778)
    with pytest.raises(hm.HMatError) as ei:
        hm.hmat_create_standard_uninit(cfg.L, cfg.d, cfg.b, cfg.r,
                                       hm._dist(nranks=2, rank=0, device=0, exchange=hm.HMAT_EXCHANGE_PEER))
    assert ei.value.status == hm.HMAT_ERR_UNSUPPORTED


def test_standard_device_generated_operator():
    """In-place device generation of the standard panels (as bench.py --config s2
    does) gives the operator the oracle sees from host-generated panels."""
    from tests.helpers import device_operator
    cfg = HConfig("stdg", d=2, L=5, b=64, r=8, adm=1, seed=779)
    h = device_operator(cfg, hm)
    try:
        x = torch.empty(cfg.N, dtype=torch.float64, device="cuda")
        hgen.dev_fill_x(cfg, 1, 0, 0, cfg.N, x.data_ptr(), cfg.N)
        y = torch.empty_like(x)
        hm.hmat_matvec(h, x, y)
        torch.cuda.synchronize()
        U, V, Dn = hgen.inputs(cfg)
        ref = oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x.cpu().numpy())
        assert_parity(y.cpu().numpy(), ref)
    finally:
        hm.hmat_destroy(h)


def test_standard_3d_leaf64_caps_pass_width():
    """3D, b = 64: 27 near-field blocks per row make wide rhs passes too big for
    shared memory; the plan caps the pass width and multi-rhs still matches."""
    cfg = HConfig("std3w", d=3, L=2, b=64, r=1, adm=1, seed=780)
    y, (U, V, Dn, x) = run_std(cfg, 5)
    assert_parity(y, oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x))


@pytest.mark.parametrize("nrhs", [1, 16])
def test_s2_full_size_sampled_rows(nrhs):
    """The bench's s2 line at full size (N = 2^20, 27 interaction slots, 55.6 GB
    of factors), in the bench's launch configuration (device-generated panels,
    default plan; 16 rhs: the tensor-core passes, 9 project slices): sampled rows
    vs the oracle's row-restricted Def 2.4 walk with on-demand factors."""
    from tests.helpers import device_operator
    cfg = hgen.EXTRA_CONFIGS["s2"]
    free, _ = torch.cuda.mem_get_info()
    if free < cfg.factor_bytes * 1.05:
        pytest.skip(f"needs {cfg.factor_bytes / 1e9:.0f} GB of device memory")
    h = device_operator(cfg, hm)
    try:
        X = torch.empty(nrhs, cfg.N, dtype=torch.float64, device="cuda")
        hgen.dev_fill_x(cfg, nrhs, 2, 0, cfg.N, X.data_ptr(), cfg.N)
        Y = torch.empty_like(X)
        hm.hmat_matvec(h, X.t(), Y.t(), nrhs)
        torch.cuda.synchronize()
        if nrhs > 1:
            assert hm.hmat_launches_per_matvec(h, nrhs) == 2
        xh = X.t().cpu().numpy()
        x, y = (xh[:, 0], Y[0]) if nrhs == 1 else (np.asfortranarray(xh), Y.t())
        n_side = 1 << cfg.L
        corner = [0, cfg.b - 1]                                      # domain corner leaf
        edge = [(n_side // 2) * cfg.b + 5]                           # a boundary leaf
        rows = np.array(sorted(set(corner + edge + [cfg.N // 2 + 17, cfg.N - 1] +
                                   list(np.random.default_rng(4).integers(0, cfg.N, 3)))))
        ref = oracle.std_rows_generated(cfg, x, rows)
        got = y.cpu().numpy()[rows]
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    finally:
        hm.hmat_destroy(h)
        torch.cuda.empty_cache()


@pytest.mark.parametrize("d,L,b,r,nrhs", [(2, 4, 4, 2, 1), (2, 3, 16, 4, 3), (1, 6, 8, 3, 2), (3, 3, 2, 1, 1),
                                          (2, 5, 16, 8, 1)])
def test_standard_literal_order_parity(d, L, b, r, nrhs):
    """hmat_create_standard_strict (Def 2.4 checked leaf first under standard
    admissibility) vs the literal-order oracle block loop, for H and H^T."""
    c = 1 << d
    N = b * c ** L
    rng = np.random.default_rng(1000 + 10 * d + L)
    M = 6 ** d - 3 ** d
    U = [rng.standard_normal((N, M * r)) / 8 for _ in range(L - 1)]
    V = [rng.standard_normal((N, M * r)) / 8 for _ in range(L - 1)]
    Dc = rng.standard_normal((N, 3 ** d * c * b)) / 8
    x = rng.uniform(-1, 1, (N, nrhs))
    h = hm.hmat_create_standard_strict(L, d, b, r, U, V, Dc)
    try:
        y = np.zeros((N, nrhs), order="F")
        hm.hmat_matvec(h, np.asfortranarray(x), y, nrhs)
        assert_parity(y, oracle.std_matvec_strict(d, L, b, r, U, V, Dc, x))
        yt = np.zeros((N, nrhs), order="F")
        hm.hmat_gemv(h, 1, 1.0, np.asfortranarray(x), 0.0, yt, nrhs)
        A = oracle.std_assemble_strict(d, L, b, r, U, V, Dc)
        assert_parity(yt, A.T @ x)
    finally:
        hm.hmat_destroy(h)


STD_DMMA = [HConfig("stdT2", d=2, L=3, b=64, r=16, adm=1, seed=790),    # W = 432: 9 project slices of 48
            HConfig("stdT2b", d=2, L=4, b=64, r=16, adm=1, seed=791),   # deeper: nodes split across CTAs
            HConfig("stdT1", d=1, L=6, b=64, r=16, adm=1, seed=792),    # W = 48: one slice
            HConfig("stdT2r", d=2, L=3, b=64, r=32, adm=1, seed=793)]   # W = 864: 9 slices of 96


@pytest.mark.parametrize("cfg", STD_DMMA, ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [5, 8, 16, 33, 64, 70])
def test_standard_tensor_core_passes(cfg, nrhs):
    """Standard admissibility on the FP64 tensor cores (one GPU, W % 16 == 0,
    64 | b): the project runs in column slices of the W = M r panel (a 2-D grid),
    scattering z through the interaction-list slot tables; the expand streams the
    3^d near-field blocks of each tile's leaf (skipping those outside the domain).
    H and H^T vs the oracle's block loops; 2 launches per pass (the tensor-core
    path ran)."""
    U, V, Dn = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, U, V, Dn)
    try:
        assert hm.hmat_launches_per_matvec(h, nrhs) == 2 * ((nrhs + 63) // 64)
        xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        yd = torch.empty_like(xd)
        hm.hmat_matvec(h, xd.t(), yd.t(), nrhs)
        yt = torch.empty_like(xd)
        hm.hmat_gemv(h, 1, 1.0, xd.t(), 0.0, yt.t(), nrhs)
        torch.cuda.synchronize()
        assert_parity(yd.t().cpu().numpy(), oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x))
        assert_parity(yt.t().cpu().numpy(), oracle.std_matvec_t(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x))
    finally:
        hm.hmat_destroy(h)


def test_standard_tensor_core_width_change_and_simt_agree():
    """Passes of different widths on one handle (64, then 8, then 64 again) and
    the SIMT kernels (HMAT_DMMA_OFF) give the same products: the z rows of slots
    outside the domain stay zero across layout changes."""
    cfg = STD_DMMA[0]
    U, V, Dn = hgen.inputs(cfg)
    h = hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, U, V, Dn)
    try:
        outs = []
        for nrhs in (64, 8, 64):
            x = hgen.xblock(cfg, nrhs=nrhs, vec=nrhs)
            xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
            yd = torch.empty_like(xd)
            hm.hmat_matvec(h, xd.t(), yd.t(), nrhs)
            torch.cuda.synchronize()
            y = yd.t().cpu().numpy()
            assert_parity(y, oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x))
            outs.append(y)
        assert np.array_equal(outs[0], outs[2])
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("cfg", STD_DMMA[:2], ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [1, 2])
def test_standard_simt_2d_r16(cfg, nrhs):
    """The SIMT path of the 2-D standard structure with r = 16, b = 64 (W = 432):
    1 rhs runs the expand's compile-time consumer shape (one row per warp, three
    near-field blocks per dense stage), 2 rhs the generic kernel.  H, H^T, and the
    two parts on their own -- the low-rank levels (hmat_matvec_parts, dense off)
    vs the oracle with the near-field blocks zeroed, the near field alone vs the
    oracle with U, V zeroed."""
    U, V, Dn = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, U, V, Dn)
    try:
        xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        outs = {}
        for name in ("full", "trans", "lowrank", "near"):
            yd = torch.full_like(xd, float("nan"))
            if name == "full":
                hm.hmat_matvec(h, xd.t(), yd.t(), nrhs)
            elif name == "trans":
                hm.hmat_gemv(h, 1, 1.0, xd.t(), 0.0, yd.t(), nrhs)
            else:
                hm.hmat_matvec_parts(h, xd.t(), yd.t(), (1 << 64) - 1 if name == "lowrank" else 0,
                                     name == "near", nrhs)
            torch.cuda.synchronize()
            outs[name] = yd.t().cpu().numpy()
        ref = lambda U_, V_, D_: oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U_, V_, D_, x)
        assert_parity(outs["full"], ref(U, V, Dn))
        assert_parity(outs["trans"], oracle.std_matvec_t(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x))
        assert_parity(outs["lowrank"], ref(U, V, np.zeros_like(Dn)))
        assert_parity(outs["near"], ref(np.zeros_like(U), np.zeros_like(V), Dn))
    finally:
        hm.hmat_destroy(h)
