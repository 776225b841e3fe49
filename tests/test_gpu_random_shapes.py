"""Seeded random sweep of shapes and right-hand-side counts through every
structure the library builds (weak, paper-strict, standard admissibility),
against the oracle: catches plan corner cases (pass widths, stage geometry,
chunked dense blocks, tensor-core eligibility) no hand-picked shape hits."""
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


def _shapes(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        d = int(rng.integers(1, 4))
        b = int(rng.choice([1, 2, 3, 5, 8, 16, 24, 64, 128]))
        r = int(rng.choice([1, 2, 3, 4, 7, 16, 32]))
        L = int(rng.integers(0, {1: 9, 2: 5, 3: 3}[d] + 1))
        N = b * (1 << d) ** L
        if N > 1 << 16 or N < 2 or ((1 << d) - 1) * r > 1024:
            continue
        nrhs = int(rng.choice([1, 2, 3, 5, 16, 64]))
        if N * nrhs > 1 << 20:
            nrhs = 1
        out.append((d, L, b, r, nrhs))
    return out


@pytest.mark.parametrize("d,L,b,r,nrhs", _shapes(24, 2026), ids=lambda v: str(v))
def test_random_weak(d, L, b, r, nrhs):
    cfg = HConfig("rnd", d=d, L=L, b=b, r=r, seed=3000 + 97 * d + 13 * L + b + r)
    U, V, D = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create(L, d, b, r, U, V, D)
    try:
        xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        yd = torch.full_like(xd, float("nan"))
        hm.hmat_matvec(h, xd.t(), yd.t(), nrhs)
        torch.cuda.synchronize()
        assert_parity(yd.t().cpu().numpy(), oracle.matvec(d, L, b, r, U, V, D, x))
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("d,L,b,r,nrhs", [s for s in _shapes(40, 77) if s[1] >= 2][:12], ids=lambda v: str(v))
def test_random_standard(d, L, b, r, nrhs):
    nrhs = min(nrhs, 3)
    cfg = HConfig("rnds", d=d, L=L, b=b, r=r, adm=1, seed=4000 + 97 * d + 13 * L + b + r)
    if cfg.slots * r > 1024:
        pytest.skip("interaction slots x rank above the kernels' limit")
    U, V, Dn = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create_standard(L, d, b, r, U, V, Dn)
    try:
        xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        yd = torch.full_like(xd, float("nan"))
        hm.hmat_matvec(h, xd.t(), yd.t(), nrhs)
        torch.cuda.synchronize()
        assert_parity(yd.t().cpu().numpy(), oracle.std_matvec(d, L, b, r, U, V, Dn, x))
    finally:
        hm.hmat_destroy(h)


@pytest.mark.parametrize("d,L,b,r,nrhs", [s for s in _shapes(40, 91) if s[1] >= 1][:10], ids=lambda v: str(v))
def test_random_strict(d, L, b, r, nrhs):
    c = 1 << d
    N = b * c ** L
    W = (c - 1) * r
    rng = np.random.default_rng(5000 + d + L + b + r)
    U = [rng.standard_normal((N, W)) / 8 for _ in range(L - 1)]
    V = [rng.standard_normal((N, W)) / 8 for _ in range(L - 1)]
    Dc = rng.standard_normal((N, c * b)) / 8
    x = rng.uniform(-1, 1, (N, nrhs))
    h = hm.hmat_create_strict(L, d, b, r, U, V, Dc)
    try:
        xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        yd = torch.full_like(xd, float("nan"))
        hm.hmat_matvec(h, xd.t(), yd.t(), nrhs)
        torch.cuda.synchronize()
        assert_parity(yd.t().cpu().numpy(), oracle.matvec_strict(d, L, b, r, U, V, Dc, x))
    finally:
        hm.hmat_destroy(h)


def _dmma_shapes(n, seed):
    """Random shapes the tensor-core path takes (W % 16 == 0 within its limits,
    64 | b), with right-hand-side counts hitting every pass width (16 / 32 / 64
    wide, ragged, several passes)."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        d = int(rng.integers(1, 4))
        c1 = (1 << d) - 1
        r = int(rng.choice([16, 32, 48, 64, 80]))
        W = c1 * r
        if W % 16 or (W % 32 == 0 and W > 224) or (W % 32 and W > 112):
            continue
        b = int(rng.choice([64, 128]))
        L = int(rng.integers(1, {1: 6, 2: 4, 3: 3}[d] + 1))
        N = b * (1 << d) ** L
        if N > 1 << 15:
            continue
        nrhs = int(rng.choice([5, 11, 16, 17, 29, 32, 40, 64, 65, 81, 100]))
        out.append((d, L, b, r, nrhs))
    return out


@pytest.mark.parametrize("d,L,b,r,nrhs", _dmma_shapes(14, 515), ids=lambda v: str(v))
def test_random_dmma(d, L, b, r, nrhs):
    cfg = HConfig("rndm", d=d, L=L, b=b, r=r, seed=5000 + 97 * d + 13 * L + b + r)
    U, V, D = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create(L, d, b, r, U, V, D)
    try:
        assert hm.hmat_launches_per_matvec(h, nrhs) == 2 * ((nrhs + 63) // 64)  # the DMMA passes
        xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        yd = torch.full_like(xd, float("nan"))
        hm.hmat_matvec(h, xd.t(), yd.t(), nrhs)
        torch.cuda.synchronize()
        assert_parity(yd.t().cpu().numpy(), oracle.matvec(d, L, b, r, U, V, D, x))
        hm.hmat_gemv(h, 1, 1.0, xd.t(), 0.0, yd.t(), nrhs)             # H^T on the same passes
        torch.cuda.synchronize()
        assert_parity(yd.t().cpu().numpy(), oracle.matvec_t(d, L, b, r, U, V, D, x))
    finally:
        hm.hmat_destroy(h)
