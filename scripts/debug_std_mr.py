"""Debug helper: P-shard standard-admissibility split-phase run with parts of
the operator zeroed; prints where the result departs from the oracle."""
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


def run(cfg, P, mode, only_level=None):
    Ug, Vg, Dg = hgen.inputs(cfg)
    if mode == "far":
        Dg = np.zeros_like(Dg)
    if mode == "near":
        Ug = [np.zeros_like(u) for u in Ug]
        Vg = [np.zeros_like(v) for v in Vg]
    if only_level is not None:
        Ug = [u if l + 1 == only_level else np.zeros_like(u) for l, u in enumerate(Ug)]
    x = hgen.xblock(cfg, nrhs=1)
    hs, xs = [], []
    for g in range(P):
        r0, r1 = g * cfg.N // P, (g + 1) * cfg.N // P
        d = hm._dist(nranks=P, rank=g, device=0, external_exchange=True)
        hs.append(hm.hmat_create_standard(cfg.L, cfg.d, cfg.b, cfg.r, [u[r0:r1] for u in Ug], [v[r0:r1] for v in Vg],
                                          Dg[r0:r1], d))
        xs.append(torch.from_numpy(np.ascontiguousarray(x[r0:r1, 0])).cuda())
    cnt = hm.hmat_exchange_size(hs[0], 1)
    ex = [torch.zeros(max(cnt, 1), dtype=torch.float64, device="cuda") for _ in range(P)]
    for g in range(P):
        hm.hmat_project(hs[g], xs[g], ex[g], 1)
    total = torch.stack(ex).sum(dim=0)
    ys = []
    for g in range(P):
        y = torch.empty_like(xs[g])
        hm.hmat_expand(hs[g], xs[g], total, y, 1)
        ys.append(y)
    torch.cuda.synchronize()
    y = torch.cat(ys).cpu().numpy()
    ref = oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, Ug, Vg, Dg, x)[:, 0]
    err = np.abs(y - ref)
    bad = np.nonzero(err > 1e-10 * np.abs(ref).max())[0]
    print(f"{cfg.name} P={P} {mode} level={only_level} cnt={cnt} rel={np.linalg.norm(y - ref) / np.linalg.norm(ref):.3e} "
          f"bad rows {len(bad)} leaves {sorted(set((bad // cfg.b).tolist()))[:20]}")
    for h in hs:
        hm.hmat_destroy(h)


if __name__ == "__main__":
    cfg = HConfig("s2d", d=2, L=4, b=8, r=3, adm=1, seed=311)
    for P in (2, 4):
        run(cfg, P, "near")
        run(cfg, P, "far")
        for l in range(2, cfg.L + 1):
            run(cfg, P, "far", l)
