"""Stress: many back-to-back matvecs (dynamic work distribution, counters re-armed
every launch) must give bitwise identical y every time."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from gen import hgen  # noqa: E402
from paper_2008_12441_b200 import hmat as hm  # noqa: E402

for name, reps in (("c2", 400), ("c3", 60), ("c5", 20)):
    cfg = hgen.CONFIGS[name]
    h = hm.hmat_create_uninit(cfg.L, cfg.d, cfg.b, cfg.r)
    r0, r1 = hm.hmat_local_rows(h)
    hgen.dev_fill_operator(cfg, lambda kind, level: hm.hmat_panel(h, kind, level), r0, r1, 0)
    n = r1 - r0
    x = torch.empty(cfg.nrhs, n, dtype=torch.float64, device="cuda")
    hgen.dev_fill_x(cfg, cfg.nrhs, 0, r0, r1, x.data_ptr(), n, 0)
    y0 = torch.empty_like(x)
    hm.hmat_matvec(h, x.t(), y0.t(), cfg.nrhs)
    y = torch.empty_like(x)
    bad = 0
    for i in range(reps):
        hm.hmat_matvec(h, x.t(), y.t(), cfg.nrhs)
        if i % 10 == 9:
            torch.cuda.synchronize()
            bad += int(not torch.equal(y, y0))
    torch.cuda.synchronize()
    print(f"{name}: {reps} matvecs, mismatching checks: {bad}", flush=True)
    assert bad == 0
    hm.hmat_destroy(h)
