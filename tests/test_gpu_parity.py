"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element, on the same seeded inputs.  Tolerance: rel l2 <= 1e-12
per right-hand side (BASELINE.json north_star) and |dy_i| <= 1e-12 max|y|."""
import itertools

import numpy as np
import pytest

from gen import hgen
from gen.hgen import CONFIGS, HConfig
from oracle import oracle
from tests.helpers import assert_parity, device_operator

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2008_12441_b200 import hmat as hm


def gpu_matvec(cfg, U, V, D, x, **kw):
    """hmat_create from host panels, device x/y, hmat_matvec."""
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        xd = torch.from_numpy(np.asfortranarray(x)).cuda() if x.ndim == 1 else \
            torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
        yd = torch.empty_like(xd) if x.ndim == 1 else torch.empty(x.shape[1], x.shape[0], dtype=torch.float64,
                                                                 device="cuda").t()
        if kw:
            hm.hmat_matvec_parts(h, xd, yd, **kw)
        else:
            hm.hmat_matvec(h, xd, yd)
        torch.cuda.synchronize()
        return yd.cpu().numpy()
    finally:
        hm.hmat_destroy(h)


def host_case(cfg, nrhs=1, vec=0):
    U, V, D = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs, vec=vec)
    if nrhs == 1:
        x = np.ascontiguousarray(x[:, 0])
    return U, V, D, x


SMALL = [HConfig(f"s{d}{L}{b}{r}", d=d, L=L, b=b, r=r, seed=1000 + 97 * d + 13 * L + 7 * b + r)
         for d, L, b, r in [
             (1, 0, 5, 1), (2, 0, 64, 3), (1, 1, 1, 1), (1, 3, 2, 2), (1, 6, 4, 3), (1, 9, 8, 5),
             (2, 1, 4, 2), (2, 2, 3, 3), (2, 3, 64, 8), (2, 4, 16, 16), (2, 3, 7, 5), (2, 5, 8, 1),
             (3, 1, 8, 4), (3, 2, 2, 2), (3, 2, 64, 32), (3, 3, 5, 3), (3, 2, 1, 7),
             (2, 3, 64, 86), (3, 2, 8, 146),  # W = 258 (> 256 consumer threads), W = 1022
         ]]


@pytest.mark.parametrize("cfg", SMALL, ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [1, 3])
def test_small_shapes(cfg, nrhs):
    """Ragged leaf sizes (odd b), ranks, depths 0..9, d = 1, 2, 3, W above the
    consumer-thread count, 1 and 3 right-hand sides."""
    U, V, D, x = host_case(cfg, nrhs)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    assert_parity(gpu_matvec(cfg, U, V, D, x), ref)


def test_c1_against_oracle_and_brute_force():
    """BASELINE configs[0] (also vs the assembled 4096 x 4096 dense matrix)."""
    cfg = CONFIGS["c1"]
    U, V, D, x = host_case(cfg)
    y = gpu_matvec(cfg, U, V, D, x)
    assert_parity(y, oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x))
    A = oracle.assemble(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D)
    assert_parity(y, oracle.dense_matvec(A, x))


@pytest.mark.parametrize("nrhs", [2, 4, 5, 8, 9, 17])
def test_multi_rhs(nrhs):
    cfg = HConfig("mr", d=3, L=3, b=64, r=8, seed=4242)  # N = 32768, W = 56
    U, V, D, x = host_case(cfg, nrhs)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    assert_parity(gpu_matvec(cfg, U, V, D, x), ref)


def test_level_parts():
    """hmat_matvec_parts reproduces the oracle's per-level pieces y_l and y_D."""
    cfg = HConfig("lp", d=2, L=5, b=16, r=4, seed=77)
    U, V, D, x = host_case(cfg)
    for mask, dense in [(0, True), (1, False), (1 << 4, False), (0b10110, False), (0, False), (0b11111, True)]:
        ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x, level_mask=mask, dense=dense)
        y = gpu_matvec(cfg, U, V, D, x, level_mask=mask, dense=dense)
        assert_parity(y, ref)


def test_c2_full_parity():
    """BASELINE configs[1] in full (N = 2^20) against the oracle's block loop."""
    cfg = CONFIGS["c2"]
    U, V, D, x = host_case(cfg)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    assert_parity(gpu_matvec(cfg, U, V, D, x), ref)


def test_host_io_misaligned_x_and_determinism():
    cfg = HConfig("io", d=2, L=4, b=64, r=16, seed=99)
    U, V, D, x = host_case(cfg, nrhs=2)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        # host numpy in/out (the e2e path)
        yh = np.zeros((cfg.N, 2), order="F")
        hm.hmat_matvec(h, np.asfortranarray(x), yh)
        assert_parity(yh, ref)
        # device, x misaligned by one double (staged internally)
        big = torch.zeros(2 * cfg.N + 1, dtype=torch.float64, device="cuda")
        xv = big[1:].view(2, cfg.N).t()
        xv.copy_(torch.from_numpy(np.asfortranarray(x)))
        yd = torch.empty(2, cfg.N, dtype=torch.float64, device="cuda").t()
        hm.hmat_matvec(h, xv, yd)
        y1 = yd.cpu().numpy()
        assert np.array_equal(y1, yh)
        # bitwise reproducible (deterministic reductions, no atomics on values)
        for _ in range(3):
            hm.hmat_matvec(h, xv, yd)
            assert np.array_equal(yd.cpu().numpy(), y1)
        assert hm.hmat_launches_per_matvec(h, 2) == 2
    finally:
        hm.hmat_destroy(h)


def test_zero_x_gives_zero():
    cfg = HConfig("z", d=3, L=2, b=64, r=4, seed=5)
    U, V, D, _ = host_case(cfg)
    y = gpu_matvec(cfg, U, V, D, np.zeros(cfg.N))
    assert np.array_equal(y, np.zeros(cfg.N))


def test_device_generator_matches_host_bitwise():
    """gen/: the device filler writes exactly the host filler's bits."""
    cfg = CONFIGS["c3"]
    for tag, level in [(hgen.TAG_U, 1), (hgen.TAG_V, 5), (hgen.TAG_D, 0)]:
        ncols = cfg.b if tag == hgen.TAG_D else cfg.W
        r0, r1 = 123456, 123456 + 700
        dev = torch.empty(r1 - r0, ncols + 2, dtype=torch.float64, device="cuda")
        hgen.dev_fill_panel(cfg, tag, level, r0, r1, dev.data_ptr(), ncols + 2)
        host = hgen.panel(cfg, tag, level, r0, r1)
        assert np.array_equal(dev[:, :ncols].cpu().numpy(), host)
    xd = torch.empty(3, 1000, dtype=torch.float64, device="cuda")
    hgen.dev_fill_x(cfg, 3, 7, 5000, 6000, xd.data_ptr(), 1000)
    assert np.array_equal(xd.cpu().numpy().T, hgen.xblock(cfg, nrhs=3, vec=7, row_begin=5000, row_end=6000))


DMMA = [HConfig("d3L2", d=3, L=2, b=64, r=32, seed=501), HConfig("d3L3", d=3, L=3, b=64, r=32, seed=502),
        HConfig("d2L3", d=2, L=3, b=64, r=32, seed=503), HConfig("d2b128", d=2, L=3, b=128, r=64, seed=504),
        # W % 32 != 0: 2 column groups x 8 rhs groups, 16-column expand chunks
        HConfig("d2r16", d=2, L=4, b=64, r=16, seed=505),    # W = 48 (the c2 / c4 shape)
        HConfig("d3r16", d=3, L=2, b=64, r=16, seed=506),    # W = 112
        HConfig("d1r16", d=1, L=6, b=64, r=16, seed=507),    # W = 16
        HConfig("d1r80", d=1, L=5, b=128, r=80, seed=508)]   # W = 80


@pytest.mark.parametrize("cfg", DMMA, ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [5, 8, 9, 16, 17, 32, 33, 64, 70, 72, 96])
def test_dmma_many_rhs(cfg, nrhs):
    """FP64 tensor-core path (nrhs >= 3, W % 16 == 0, 64 | b): passes of 64
    right-hand sides, the last one 8, 16 or 32 wide when at most 8 / 16 / 32
    remain (5 | 8, 9 | 16, 17, 32 | 70 = 64 + 6, 72 = 64 + 8 | 96 = 64 + 32),
    ragged passes, vs the oracle."""
    U, V, D, x = host_case(cfg, nrhs)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        assert hm.hmat_launches_per_matvec(h, nrhs) == 2 * ((nrhs + 63) // 64)  # the DMMA passes ran
    finally:
        hm.hmat_destroy(h)
    assert_parity(gpu_matvec(cfg, U, V, D, x), ref)



@pytest.mark.parametrize("cfg", [DMMA[0], DMMA[4], DMMA[6], DMMA[7]], ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [1, 2, 3, 4])
def test_dmma_8wide_pass_few_rhs(cfg, nrhs, monkeypatch):
    """The 8-wide tensor-core pass (one N-tile: fragment-major Zt of one double
    per lane) serving 1..4 rhs when the threshold is lowered (HMAT_DMMA_MIN)."""
    monkeypatch.setenv("HMAT_DMMA_MIN", "1")
    U, V, D, x = host_case(cfg, nrhs)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        assert hm.hmat_plan_query(cfg.L, cfg.d, cfg.b, cfg.r).dmma_ok[3] == 1
        y = np.zeros((cfg.N, nrhs), order="F")
        hm.hmat_matvec(h, np.asfortranarray(x.reshape(cfg.N, nrhs)), y, nrhs)
        assert_parity(y, ref.reshape(cfg.N, nrhs))
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("nw", ["2", "6"])
@pytest.mark.parametrize("nrhs", [3, 8, 11])
def test_dmma_8wide_project_warp_splits(nw, nrhs, monkeypatch):
    """The 8-wide project's CTA shapes at W = 48 (HMAT_DMMA8_NW: 2 warps x 24
    columns, 6 x 8; the default 3 x 16 runs everywhere else), with 3 and 8 rhs
    (one 8-wide pass) and 11 (one 16-wide pass, unaffected)."""
    monkeypatch.setenv("HMAT_DMMA8_NW", nw)
    cfg = HConfig("nw48", d=2, L=4, b=64, r=16, seed=91)   # W = 48
    U, V, D, x = host_case(cfg, nrhs)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        y = np.zeros((cfg.N, nrhs), order="F")
        hm.hmat_matvec(h, np.asfortranarray(x.reshape(cfg.N, nrhs)), y, nrhs)
        assert_parity(y, ref.reshape(cfg.N, nrhs))
    finally:
        hm.hmat_destroy(h)


def _dev_cols(x):
    """host (N,) / (N, k) array -> device tensor with the same column-major layout."""
    if x.ndim == 1:
        return torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()


@pytest.mark.parametrize("cfg", [HConfig("g1", d=2, L=3, b=16, r=4, seed=81), HConfig("g2", d=3, L=2, b=7, r=3, seed=82),
                                 HConfig("g3", d=1, L=5, b=4, r=2, seed=83)], ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [1, 3])
def test_gemv_alpha_beta_and_transpose(cfg, nrhs):
    """hmat_gemv: y = alpha op(H) x + beta y for op = H, H^T;
    beta = 0 must not read y (NaN in y stays out of the result)."""
    U, V, D, x = host_case(cfg, nrhs)
    Hx = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    HTx = oracle.matvec_t(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    rng = np.random.default_rng(5)
    y0 = rng.standard_normal(x.shape)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        for trans, ref in ((0, Hx), (1, HTx)):
            yd = _dev_cols(y0)
            hm.hmat_gemv(h, trans, -1.5, _dev_cols(x), 0.25, yd)
            assert_parity(yd.cpu().numpy(), -1.5 * ref + 0.25 * y0)
            yn = _dev_cols(np.full(x.shape, np.nan))
            hm.hmat_gemv(h, trans, 2.0, _dev_cols(x), 0.0, yn)
            assert_parity(yn.cpu().numpy(), 2.0 * ref)
        # host y with beta != 0 is read and written
        yh = np.asfortranarray(y0.copy()) if y0.ndim > 1 else y0.copy()
        hm.hmat_gemv(h, 1, 1.0, np.asfortranarray(x) if x.ndim > 1 else x, 1.0, yh)
        assert_parity(yh, HTx + y0)
    finally:
        hm.hmat_destroy(h)


def test_adjoint_identity_c2_and_dmma():
    """<y', H x> = <H^T y', x> at C2 size (SIMT path) and on a DMMA-eligible
    shape with 64 right-hand sides (tensor-core path)."""
    for cfg, nrhs in ((CONFIGS["c2"], 1), (HConfig("adj", d=3, L=3, b=64, r=32, seed=85), 64)):
        h = device_operator(cfg, hm)
        try:
            n = cfg.N
            X = torch.empty(nrhs, n, dtype=torch.float64, device="cuda")
            Yp = torch.empty_like(X)
            hgen.dev_fill_x(cfg, nrhs, 0, 0, n, X.data_ptr(), n)
            hgen.dev_fill_x(cfg, nrhs, 1, 0, n, Yp.data_ptr(), n)
            HX = torch.empty_like(X)
            HTY = torch.empty_like(X)
            hm.hmat_gemv(h, 0, 1.0, X.t(), 0.0, HX.t())
            hm.hmat_gemv(h, 1, 1.0, Yp.t(), 0.0, HTY.t())
            lhs = (Yp * HX).sum(dim=1)
            rhs = (HTY * X).sum(dim=1)
            scale = (Yp.abs() * HX.abs()).sum(dim=1)
            assert torch.all((lhs - rhs).abs() <= 1e-12 * scale)
        finally:
            hm.hmat_destroy(h)
            torch.cuda.empty_cache()


@pytest.mark.parametrize("d,L,b,r", [(2, 3, 16, 4), (3, 2, 8, 2), (1, 4, 2, 3), (2, 1, 5, 2),
                                     (2, 3, 64, 4), (3, 2, 16, 2), (1, 5, 64, 3)])  # leaf 256 / 128 / 128: chunked dense
def test_strict_structure(d, L, b, r):
    """hmat_create_strict (Def 2.4 read literally: leaf-parent diagonal blocks
    dense) vs the oracle's strict block loop."""
    c = 1 << d
    N = b * c ** L
    W = (c - 1) * r
    rng = np.random.default_rng(90 + L)
    U = [rng.standard_normal((N, W)) / 8 for _ in range(L - 1)]
    V = [rng.standard_normal((N, W)) / 8 for _ in range(L - 1)]
    Dc = rng.standard_normal((N, c * b)) / 8
    x = rng.uniform(-1, 1, (N, 2))
    ref = oracle.matvec_strict(d, L, b, r, U, V, Dc, x)
    h = hm.hmat_create_strict(L, d, b, r, U, V, Dc)
    try:
        y = _dev_cols(np.zeros((N, 2)))
        hm.hmat_matvec(h, _dev_cols(x), y)
        assert_parity(y.cpu().numpy(), ref)
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("chunk,pdyn", [("0", "0"), ("1", "1"), ("3", "1"), ("1", "0")])
def test_expand_work_distribution_and_rearm(chunk, pdyn, monkeypatch):
    """Work distribution: expand's static item ranges (HMAT_EXPAND_CHUNK=0) or
    dynamic chunks of 1 / 3 items, project's last level static or in dynamic
    node chunks (HMAT_PROJECT_DYN), give the same y, for several matvecs in a
    row on one handle (the counters are re-armed by the last CTA of every
    launch)."""
    monkeypatch.setenv("HMAT_EXPAND_CHUNK", chunk)
    monkeypatch.setenv("HMAT_PROJECT_DYN", pdyn)
    cfg = HConfig("chunks", d=2, L=6, b=16, r=4, seed=1201)   # 4096 items of 16 rows: ~14 per CTA
    U, V, D = hgen.inputs(cfg)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        for v in range(3):
            x = np.ascontiguousarray(hgen.xblock(cfg, nrhs=1, vec=v)[:, 0])
            xd = torch.from_numpy(x).cuda()
            yd = torch.full_like(xd, float("nan"))
            hm.hmat_matvec(h, xd, yd)
            torch.cuda.synchronize()
            assert_parity(yd.cpu().numpy(), oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x))
    finally:
        hm.hmat_destroy(h)


def test_strict_chunked_dense_adjoint():
    """Paper-strict structure with leaf 256 (the dense block travels in 64-column
    chunks): <y', H x> = <H^T y', x> with both products on the GPU."""
    d, L, b, r = 2, 4, 64, 4
    c = 1 << d
    N = b * c ** L
    W = (c - 1) * r
    rng = np.random.default_rng(1301)
    U = [rng.standard_normal((N, W)) / 8 for _ in range(L - 1)]
    V = [rng.standard_normal((N, W)) / 8 for _ in range(L - 1)]
    Dc = rng.standard_normal((N, c * b)) / 8
    h = hm.hmat_create_strict(L, d, b, r, U, V, Dc)
    try:
        x = torch.from_numpy(rng.standard_normal(N)).cuda()
        yp = torch.from_numpy(rng.standard_normal(N)).cuda()
        hx, hty = torch.empty_like(x), torch.empty_like(x)
        hm.hmat_gemv(h, 0, 1.0, x, 0.0, hx)
        hm.hmat_gemv(h, 1, 1.0, yp, 0.0, hty)
        torch.cuda.synchronize()
        lhs, rhs = float(yp @ hx), float(hty @ x)
        assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    finally:
        hm.hmat_destroy(h)


def test_host_async_streaming_mode():
    """hmat_set_host_async: host-pointer matvecs return once enqueued, copies
    overlap neighbouring calls; after hmat_synchronize every y is right (the
    alternating staging buffers are never reused too early), also for 3 rhs
    and GEMV with beta != 0 (y is an input)."""
    cfg = HConfig("async", d=2, L=5, b=16, r=4, seed=1401)
    U, V, D = hgen.inputs(cfg)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        hm.hmat_set_host_async(h, True)
        xs = [torch.from_numpy(np.ascontiguousarray(hgen.xblock(cfg, nrhs=1, vec=v)[:, 0])).pin_memory()
              for v in range(5)]
        ys = [torch.full((cfg.N,), float("nan"), dtype=torch.float64).pin_memory() for _ in range(5)]
        for x, y in zip(xs, ys):
            hm.hmat_matvec(h, x, y)
        x3 = torch.from_numpy(np.ascontiguousarray(hgen.xblock(cfg, nrhs=3, vec=7).T)).pin_memory()
        y3 = torch.full_like(x3, float("nan")).pin_memory()
        hm.hmat_matvec(h, x3.t(), y3.t())
        y0 = np.random.default_rng(5).standard_normal(cfg.N)
        yb = torch.from_numpy(y0.copy()).pin_memory()
        hm.hmat_gemv(h, 0, 2.0, xs[0], -1.0, yb)
        hm.hmat_synchronize(h)
        for x, y in zip(xs, ys):
            assert_parity(y.numpy(), oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x.numpy()))
        assert_parity(y3.t().numpy(), oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x3.t().numpy()))
        assert_parity(yb.numpy(), 2.0 * oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, xs[0].numpy()) - y0)
        hm.hmat_set_host_async(h, False)            # back to blocking: returns with y home
        yy = torch.empty(cfg.N, dtype=torch.float64).pin_memory()
        hm.hmat_matvec(h, xs[1], yy)
        assert_parity(yy.numpy(), ys[1].numpy())
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("chunks", ["1", "3", "8"])
@pytest.mark.parametrize("nrhs", [1, 9, 70])
def test_host_y_row_chunks_bitwise(chunks, nrhs, monkeypatch):
    """A host y leaves in row chunks of whole leaves while the expand computes
    the next ones (HMAT_Y_CHUNKS; the expand runs once per chunk over an item
    range, from 4 MB of y): y is bit-identical to the device-pointer product, for
    1 rhs (0.5 MB: one piece) and the tensor-core kernels (9: one 16-wide pass,
    70: a 64- and an 8-wide pass), in the blocking and the streaming mode."""
    monkeypatch.setenv("HMAT_Y_CHUNKS", chunks)
    cfg = HConfig("ych", d=2, L=5, b=64, r=16, seed=1402)   # 1024 leaves: y >= 4 MB from 9 rhs
    U, V, D = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        yd = torch.empty_like(xd)
        hm.hmat_matvec(h, xd.t(), yd.t(), nrhs)
        torch.cuda.synchronize()
        ref = yd.t().cpu().numpy()
        xh = torch.from_numpy(np.ascontiguousarray(x.T)).pin_memory()
        yh = torch.full_like(xh, float("nan")).pin_memory()
        hm.hmat_matvec(h, xh.t(), yh.t(), nrhs)                       # blocking
        assert np.array_equal(yh.t().numpy(), ref)
        hm.hmat_set_host_async(h, True)                                # streaming
        ys = [torch.full_like(xh, float("nan")).pin_memory() for _ in range(3)]
        for y in ys:
            hm.hmat_matvec(h, xh.t(), y.t(), nrhs)
        hm.hmat_synchronize(h)
        for y in ys:
            assert np.array_equal(y.t().numpy(), ref)
        assert_parity(ref, oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x))
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("snake", ["0", "1"])
def test_project_stream_direction(snake, monkeypatch):
    """Project's per-level stream direction (HMAT_PROJECT_SNAKE): backwards even
    levels reorder each node's row sums and the CTA partials' flushes; y stays
    within tolerance and bitwise reproducible, with nodes cut by CTA ranges."""
    monkeypatch.setenv("HMAT_PROJECT_SNAKE", snake)
    monkeypatch.setenv("HMAT_PROJECT_DYN", "0")
    cfg = HConfig("sn", d=2, L=5, b=16, r=4, seed=610)   # 1024 leaves: coarse nodes span many CTAs
    U, V, D, x = host_case(cfg, nrhs=3)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    y1 = gpu_matvec(cfg, U, V, D, x)
    assert_parity(y1, ref)
    assert np.array_equal(gpu_matvec(cfg, U, V, D, x), y1)


def test_host_async_pipeline_bitwise_at_c2_size():
    """The streaming host mode at C2 size (copies and kernels of neighbouring
    calls overlap for real): a run of calls mixing y = Hx and y = 2Hx - y (y an
    input, read from host staging that an earlier call's copy-out may still be
    using), distinct host buffers, equals the blocking device-pointer results
    bit for bit."""
    cfg = CONFIGS["c2"]
    h = device_operator(cfg, hm)
    try:
        n, calls = cfg.N, 8
        X = torch.empty(calls, n, dtype=torch.float64, device="cuda")
        for v in range(calls):
            hgen.dev_fill_x(cfg, 1, v, 0, n, X[v].data_ptr(), n)
        Y0 = torch.randn(calls, n, dtype=torch.float64, generator=torch.Generator().manual_seed(9)).cuda()
        want = []
        for v in range(calls):                      # blocking, device pointers
            yv = Y0[v].clone()
            if v % 2:
                hm.hmat_gemv(h, 0, 2.0, X[v], -1.0, yv)
            else:
                hm.hmat_matvec(h, X[v], yv)
            want.append(yv.cpu())
        xh = [X[v].cpu().pin_memory() for v in range(calls)]
        yh = [Y0[v].cpu().pin_memory() for v in range(calls)]
        torch.cuda.synchronize()
        hm.hmat_set_host_async(h, True)
        for v in range(calls):
            if v % 2:
                hm.hmat_gemv(h, 0, 2.0, xh[v], -1.0, yh[v])
            else:
                hm.hmat_matvec(h, xh[v], yh[v])
        hm.hmat_synchronize(h)
        hm.hmat_set_host_async(h, False)
        for v in range(calls):
            assert torch.equal(yh[v], want[v]), f"call {v}"
    finally:
        hm.hmat_destroy(h)
        torch.cuda.empty_cache()


@pytest.mark.parametrize("nrhs", [1, 64])
def test_cuda_graph_capture_and_replay(nrhs):
    """A matvec is capture-safe (P = 1): warmed up once (lazy buffers), captured
    into a CUDA graph on the capturing stream (hmat_set_stream), replayed on new x
    -- same bits as direct calls (the dynamic work counters re-arm inside the
    kernels, so replays need no host work)."""
    cfg = HConfig("graph", d=2, L=4, b=64, r=16, seed=1601)           # W = 48: nrhs 64 takes DMMA
    U, V, D = hgen.inputs(cfg)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        xs = [torch.from_numpy(np.ascontiguousarray(hgen.xblock(cfg, nrhs=nrhs, vec=v).T)).cuda() for v in range(3)]
        x = torch.empty_like(xs[0])
        y = torch.empty_like(xs[0])
        s = torch.cuda.Stream()
        hm.hmat_set_stream(h, s.cuda_stream)
        with torch.cuda.stream(s):
            x.copy_(xs[0])
            hm.hmat_matvec(h, x.t(), y.t(), nrhs)                      # warm-up: lazy allocations
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            hm.hmat_matvec(h, x.t(), y.t(), nrhs)
        for v in (1, 2, 1):
            x.copy_(xs[v])
            g.replay()
            torch.cuda.synchronize()
            want = torch.empty_like(y)
            with torch.cuda.stream(s):
                hm.hmat_matvec(h, xs[v].t(), want.t(), nrhs)
            s.synchronize()
            assert torch.equal(y, want)
        ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, xs[1].t().cpu().numpy())
        x.copy_(xs[1])
        g.replay()
        torch.cuda.synchronize()
        assert_parity(y.t().cpu().numpy(), ref)
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("cfg", [HConfig("lp1", d=2, L=3, b=64, r=8, seed=1701),     # c1's shape
                                 HConfig("lp2", d=3, L=2, b=16, r=4, seed=1702),     # nodes over many CTAs
                                 HConfig("lp3", d=1, L=6, b=8, r=3, seed=1703)], ids=lambda c: c.name)
def test_project_level_parallel_mode(cfg, monkeypatch):
    """Small operators: project in level-parallel mode (one stage of one level per
    CTA, HMAT_PROJECT_LPAR) equals the oracle, the per-level pieces too (a
    subset of active levels), and the default split bit for bit (same CTA
    partition of each level when every level fits the grid)."""
    U, V, D, x = host_case(cfg, nrhs=3)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    monkeypatch.setenv("HMAT_PROJECT_LPAR", "1")
    y1 = gpu_matvec(cfg, U, V, D, x)
    assert_parity(y1, ref)
    mask = 0b101 if cfg.L >= 3 else 0b11
    assert_parity(gpu_matvec(cfg, U, V, D, x, level_mask=mask, dense=False),
                  oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x, level_mask=mask, dense=False))
    monkeypatch.setenv("HMAT_PROJECT_LPAR", "0")
    assert np.array_equal(gpu_matvec(cfg, U, V, D, x), y1)


@pytest.mark.parametrize("pdl", ["0", "1", "2"])
def test_power_iteration_chains_products(pdl, monkeypatch):
    """x_{k+1} = H x_k with the buffers swapped between calls and no host sync:
    each product's project reads what the previous expand wrote (the hazard the
    programmatic dependent launches must respect, HMAT_PDL).  Every setting gives
    the same bits, and the oracle's iterates."""
    monkeypatch.setenv("HMAT_PDL", pdl)
    cfg = HConfig("pw", d=2, L=3, b=64, r=8, seed=1801)            # c1's shape (level-parallel project)
    U, V, D = hgen.inputs(cfg)
    x0 = hgen.xblock(cfg, nrhs=1)[:, 0]
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        a = torch.from_numpy(x0.copy()).cuda()
        b = torch.empty_like(a)
        iters = 12
        for k in range(iters):
            hm.hmat_matvec(h, a, b)
            a, b = b, a
            a.mul_(1.0 / 8.0)                                          # keep the iterates bounded (a torch kernel in between)
        torch.cuda.synchronize()
        got = a.cpu().numpy()
    finally:
        hm.hmat_destroy(h)
    ref = x0.copy()
    for k in range(iters):
        ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, ref) / 8.0
    assert np.linalg.norm(got - ref) <= 1e-11 * np.linalg.norm(ref)
    tag = f"pw_{pdl}"
    test_power_iteration_chains_products.results = getattr(test_power_iteration_chains_products, "results", {})
    test_power_iteration_chains_products.results[tag] = got
    if len(test_power_iteration_chains_products.results) == 3:
        vals = list(test_power_iteration_chains_products.results.values())
        assert all(np.array_equal(v, vals[0]) for v in vals)


def test_power_iteration_back_to_back_products(monkeypatch):
    """The same chain with nothing between the products (expand k -> project k+1
    directly: the programmatic launch edge itself), iterates compared bit for
    bit with HMAT_PDL=0."""
    cfg = HConfig("pw2", d=2, L=3, b=64, r=8, seed=1802)
    U, V, D = hgen.inputs(cfg)
    x0 = hgen.xblock(cfg, nrhs=1)[:, 0] / 64.0
    outs = []
    for pdl in ("0", "2"):
        monkeypatch.setenv("HMAT_PDL", pdl)
        h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
        try:
            a = torch.from_numpy(x0.copy()).cuda()
            b = torch.empty_like(a)
            for k in range(10):
                hm.hmat_matvec(h, a, b)
                a, b = b, a
            torch.cuda.synchronize()
            outs.append(a.cpu().numpy())
        finally:
            hm.hmat_destroy(h)
    assert np.array_equal(outs[0], outs[1])
    ref = x0.copy()
    for k in range(10):
        ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, ref)
    assert np.linalg.norm(outs[1] - ref) <= 1e-11 * np.linalg.norm(ref)


@pytest.mark.parametrize("width", [8, 16])
@pytest.mark.parametrize("mask", [1 << 2, 1 << 4, 0b10100, 0b01011])
def test_dmma_project_level_chunks_masked(mask, width, monkeypatch):
    """Level-interleaved chunks with a level mask (hmat_matvec_parts): a single
    active level (its next (chunk, level) is itself, whose running sums of the
    chunk are saved only at the level's end) and non-adjacent levels; the
    tensor-core project loads the next level's sums one level ahead.  Parity with
    the oracle's parts and bit-identical to the unchunked order."""
    cfg = HConfig("ckm", d=2, L=5, b=64, r=16, seed=515)                              # W = 48
    nrhs = 8 if width == 8 else 13
    U, V, D, x = host_case(cfg, nrhs)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x, level_mask=mask, dense=False)
    outs = []
    for ch in (3, 0):
        monkeypatch.setenv("HMAT_DMMA_PCHUNK" if width == 8 else "HMAT_DMMA_PCHUNK16", str(ch))
        outs.append(gpu_matvec(cfg, U, V, D, x, level_mask=mask, dense=False))
    assert_parity(outs[0], ref)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("cfg", [HConfig("ck48", d=2, L=5, b=64, r=16, seed=511),    # W = 48
                                 HConfig("ck16", d=1, L=11, b=64, r=16, seed=512),   # W = 16
                                 HConfig("ck80", d=1, L=10, b=128, r=80, seed=513),  # W = 80
                                 HConfig("ck112", d=3, L=3, b=64, r=16, seed=514)],  # W = 112
                         ids=lambda c: c.name)
@pytest.mark.parametrize("chunk", [1, 3, 7])
@pytest.mark.parametrize("width", [8, 16])
def test_dmma_project_level_chunks(cfg, chunk, width, monkeypatch):
    """8- and 16-wide passes interleave the levels in chunks of HMAT_DMMA_PCHUNK /
    HMAT_DMMA_PCHUNK16 stages of each CTA's range, carrying the running sums between chunks (kernels_dmma.cu);
    small chunks put chunk boundaries inside nodes of every level.  The result is
    the oracle's and bit-identical to the unchunked level order (each level's
    stages are summed in the same order)."""
    nrhs = 8 if width == 8 else 13  # one 8-wide / one 16-wide pass
    U, V, D, x = host_case(cfg, nrhs)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    outs = []
    for ch in (chunk, 0):
        monkeypatch.setenv("HMAT_DMMA_PCHUNK" if width == 8 else "HMAT_DMMA_PCHUNK16", str(ch))
        h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
        try:
            y = np.zeros((cfg.N, nrhs), order="F")
            hm.hmat_matvec(h, np.asfortranarray(x), y, nrhs)
            outs.append(y)
        finally:
            hm.hmat_destroy(h)
    assert_parity(outs[0], ref)
    assert np.array_equal(outs[0], outs[1])
