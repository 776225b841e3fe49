"""Per-CTA load balance of the project / expand kernels (hmat_cta_trace).

    python scripts/cta_trace.py c5 [d=3,L=4,b=64,r=32,nrhs=64 ...]

Runs warm-up matvecs, then one traced matvec, and prints for each kernel the
spread of CTA start / end times relative to the kernel's first CTA start, the
slowest CTAs (with their SM ids) and how many CTAs shared an SM.
"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from gen import hgen  # noqa: E402
from paper_2008_12441_b200 import hmat as hm  # noqa: E402
from scripts.kernel_sweep import parse_cfg  # noqa: E402


def report(name, recs):
    recs = [r for r in recs if r[1] > 0]
    if not recs:
        print(f"  {name}: no records")
        return
    t0 = min(r[0] for r in recs)
    starts = sorted((r[0] - t0) / 1e3 for r in recs)
    ends = sorted((r[1] - t0) / 1e3 for r in recs)
    durs = sorted((r[1] - r[0]) / 1e3 for r in recs)
    q = lambda v, f: v[min(len(v) - 1, int(f * len(v)))]  # noqa: E731
    print(f"  {name}: {len(recs)} CTAs, kernel span {ends[-1]:.1f} us | start max {starts[-1]:.1f} us | "
          f"end min/med/p90/max {ends[0]:.1f}/{q(ends, .5):.1f}/{q(ends, .9):.1f}/{ends[-1]:.1f} us | "
          f"dur min/med/max {durs[0]:.1f}/{q(durs, .5):.1f}/{durs[-1]:.1f} us | "
          f"idle {1 - sum(durs) / (len(durs) * ends[-1]):.1%} of CTA-slots")
    sm_end = collections.defaultdict(float)
    for r in recs:
        sm_end[r[2]] = max(sm_end[r[2]], (r[1] - t0) / 1e3)
    se = sorted(sm_end.values())
    print(f"  {name}: per-SM last end min/med/max {se[0]:.1f}/{q(se, .5):.1f}/{se[-1]:.1f} us "
          f"(SM-level idle {1 - sum(se) / (len(se) * se[-1]):.1%})")
    per_sm = collections.Counter(r[2] for r in recs)
    print(f"  {name}: {len(per_sm)} SMs used, CTAs per SM {sorted(collections.Counter(per_sm.values()).items())}")
    slow = sorted(enumerate(recs), key=lambda e: e[1][1] - e[1][0], reverse=True)[:6]
    print("  slowest: " + ", ".join(f"cta {b} sm {r[2]} start {(r[0] - t0) / 1e3:.1f} dur {(r[1] - r[0]) / 1e3:.1f} us"
                                     for b, r in slow))


def run(cfg):
    h = (hm.hmat_create_standard_uninit if cfg.adm else hm.hmat_create_uninit)(cfg.L, cfg.d, cfg.b, cfg.r)
    try:
        r0, r1 = hm.hmat_local_rows(h)
        hgen.dev_fill_operator(cfg, lambda kind, level: hm.hmat_panel(h, kind, level), r0, r1, 0)
        n = r1 - r0
        x = torch.empty(cfg.nrhs, n, dtype=torch.float64, device="cuda")
        hgen.dev_fill_x(cfg, cfg.nrhs, 0, r0, r1, x.data_ptr(), n, 0)
        y = torch.empty_like(x)
        for _ in range(3):
            hm.hmat_matvec(h, x.t(), y.t(), cfg.nrhs)
        hm.hmat_cta_trace(h, True)
        hm.hmat_matvec(h, x.t(), y.t(), cfg.nrhs)
        print(f"{cfg.name}:")
        report("project", hm.hmat_cta_trace_read(h, 0))
        report("expand ", hm.hmat_cta_trace_read(h, 1))
        hm.hmat_cta_trace(h, False)
    finally:
        hm.hmat_destroy(h)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    for spec in sys.argv[1:] or ["c2"]:
        run(parse_cfg(spec))
