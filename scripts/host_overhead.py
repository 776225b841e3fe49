"""Host cost of one hmat_matvec call (enqueue only) vs its GPU time, on small configs."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from gen import hgen  # noqa: E402
from paper_2008_12441_b200 import hmat as hm  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2"]:
    cfg = {**hgen.CONFIGS, **hgen.EXTRA_CONFIGS}[name]
    h = hm.hmat_create_uninit(cfg.L, cfg.d, cfg.b, cfg.r)
    r0, r1 = hm.hmat_local_rows(h)
    hgen.dev_fill_operator(cfg, lambda kind, level: hm.hmat_panel(h, kind, level), r0, r1, 0)
    x = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
    hgen.dev_fill_x(cfg, 1, 0, r0, r1, x.data_ptr(), r1 - r0, 0)
    y = torch.empty_like(x)
    for _ in range(20):
        hm.hmat_matvec(h, x, y)
    torch.cuda.synchronize()
    n = 2000 if name == "c1" else 200
    t0 = time.perf_counter()
    for _ in range(n):
        hm.hmat_matvec(h, x, y)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host enqueue {1e6 * (t1 - t0) / n:.1f} us/call, wall incl. GPU {1e6 * (t2 - t0) / n:.1f} us/call")
    hm.hmat_destroy(h)
