"""Per-level kernel timing: project/expand GB/s when only one level (or only the
dense leaf blocks) is active, via hmat_matvec_parts.  usage: level_profile.py c4"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from gen import hgen  # noqa: E402
from paper_2008_12441_b200 import hmat as hm  # noqa: E402

cfg = {**hgen.CONFIGS, **hgen.EXTRA_CONFIGS}[sys.argv[1]]
reps = 10
h = (hm.hmat_create_standard_uninit if cfg.adm else hm.hmat_create_uninit)(cfg.L, cfg.d, cfg.b, cfg.r)
r0, r1 = hm.hmat_local_rows(h)
hgen.dev_fill_operator(cfg, lambda kind, level: hm.hmat_panel(h, kind, level), r0, r1, 0)
n = r1 - r0
x = torch.empty(n, dtype=torch.float64, device="cuda")
hgen.dev_fill_x(cfg, 1, 0, r0, r1, x.data_ptr(), n, 0)
y = torch.empty_like(x)
torch.cuda.synchronize()
for _ in range(int(os.environ.get("WARM", "0"))):  # e.g. reach the sustained power cap first
    hm.hmat_matvec(h, x, y)
cases = [(f"level {l}", 1 << (l - 1), False) for l in range(1, cfg.L + 1)] + [("dense", 0, True), ("no last", (1 << (cfg.L - 1)) - 1, False), ("all", (1 << cfg.L) - 1, True)]
for name, mask, dense in cases:
    for _ in range(2):
        hm.hmat_matvec_parts(h, x, y, mask, dense)
    hm.hmat_profile(h, True)
    hm.hmat_profile_read(h)
    for _ in range(reps):
        hm.hmat_matvec_parts(h, x, y, mask, dense)
    prof = hm.hmat_profile_read(h)
    hm.hmat_profile(h, False)
    nl = bin(mask).count("1")
    pb = 8 * n * cfg.W * nl
    eb = 8 * n * (cfg.W * nl + (cfg.dcols if dense else 0))
    pm = prof["project"][0] / max(1, prof["project"][1])
    em = prof["expand"][0] / max(1, prof["expand"][1])
    print(f"{cfg.name} {name:9s} project {pm:8.3f} ms {pb / max(pm, 1e-9) / 1e6:6.0f} GB/s | "
          f"expand {em:8.3f} ms {eb / max(em, 1e-9) / 1e6:6.0f} GB/s", flush=True)
hm.hmat_destroy(h)
