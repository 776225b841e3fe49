"""Small products through every kernel family, each checked against the oracle
(a quick end-to-end check after a kernel change; compute-sanitizer is not
available on the GPU pool):

    python scripts/small_families.py

weak 1 rhs (compile-time shapes W = 48 / 224), 2 rhs (generic SIMT), 5 / 12 / 40
rhs (tensor-core passes 8 / 16 / 64 wide, plain-product variant), a level-masked
part (general variant); standard 1 rhs (W = 432 shape), 16 rhs on the tensor cores,
and P = 2 shards of it through the split-phase calls.  Results are checked against
the oracle (test infrastructure) so a silent corruption also fails."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import hgen  # noqa: E402
from gen.hgen import HConfig  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2008_12441_b200 import hmat as hm  # noqa: E402


def check(y, ref, what):
    err = np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-300)
    print(f"{what}: rel l2 {err:.2e}")
    assert err < 1e-12, what


def weak(cfg, nrhs, mask=None):
    U, V, D = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        yd = torch.empty_like(xd)
        if mask is None:
            hm.hmat_matvec(h, xd.t(), yd.t(), nrhs)
            ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
        else:
            hm.hmat_matvec_parts(h, xd.t(), yd.t(), mask, False, nrhs)
            ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x, level_mask=mask, dense=False)
        torch.cuda.synchronize()
        check(yd.t().cpu().numpy(), ref, f"weak {cfg.name} nrhs={nrhs} mask={mask}")
    finally:
        hm.hmat_destroy(h)


def standard(cfg, nrhs, P=1):
    U, V, Dn = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs)
    ref = oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x)
    if P == 1:
        h = hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, U, V, Dn)
        try:
            xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
            yd = torch.empty_like(xd)
            hm.hmat_matvec(h, xd.t(), yd.t(), nrhs)
            torch.cuda.synchronize()
            check(yd.t().cpu().numpy(), ref, f"standard {cfg.name} nrhs={nrhs}")
        finally:
            hm.hmat_destroy(h)
        return
    hs, xs = [], []
    try:
        for g in range(P):
            r0, r1 = g * cfg.N // P, (g + 1) * cfg.N // P
            Ug, Vg, Dg = hgen.inputs(cfg, r0, r1)
            hs.append(hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, Ug, Vg, Dg,
                                              hm._dist(nranks=P, rank=g, device=0, external_exchange=True)))
            xs.append(torch.from_numpy(np.ascontiguousarray(x[r0:r1].T)).cuda())
        cnt = hm.hmat_exchange_size(hs[0], nrhs)
        ex = [torch.zeros(max(cnt, 1), dtype=torch.float64, device="cuda") for _ in range(P)]
        for g in range(P):
            hm.hmat_project(hs[g], xs[g].t(), ex[g], nrhs)
        torch.cuda.synchronize()
        total = torch.stack(ex).sum(dim=0)
        ys = []
        for g in range(P):
            y = torch.empty_like(xs[g])
            hm.hmat_expand(hs[g], xs[g].t(), total, y.t(), nrhs)
            ys.append(y)
        torch.cuda.synchronize()
        check(torch.cat(ys, dim=1).t().cpu().numpy(), ref, f"standard {cfg.name} nrhs={nrhs} P={P}")
    finally:
        for h in hs:
            hm.hmat_destroy(h)


if __name__ == "__main__":
    w48 = HConfig("w48", d=2, L=3, b=64, r=16, seed=601)     # W = 48
    w224 = HConfig("w224", d=3, L=2, b=64, r=32, seed=602)   # W = 224
    for cfg in (w48, w224):
        for nrhs in (1, 2, 5, 12, 40):
            weak(cfg, nrhs)
    weak(w48, 5, mask=0b101)
    s2 = HConfig("s2s", d=2, L=3, b=64, r=16, adm=1, seed=603)  # W = 432
    standard(s2, 1)
    standard(s2, 16)
    standard(s2, 16, P=2)
    standard(s2, 1, P=2)
    print("ok")
