"""Per-rank work of a P-GPU product, measured on the one GPU of the box.

    python scripts/shard_times.py [c4] [P ...]      (default: c4, P = 1 2 4 8)

For each P, rank g's shard of the operator (its Morton rows [g N/P, (g+1) N/P) of
every panel, built exactly as bench.py's rank g builds it, with
a caller-provided exchange) runs hmat_project -> hmat_expand back to back with
CUDA events on its stream: the time rank g spends in its kernels per product,
with nothing skipped except the cross-GPU sum of the packed exchange buffer
(whose bytes are printed: 7.7 KB for 2D at P = 8).  Ranks 0 and P-1 are timed
(the first and last shards differ in which coarse-level nodes they split).  The
exchange itself needs P GPUs and is NOT measured here; a P-GPU step takes
max over ranks of (kernels + exchange).  One JSON line per (P, rank).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from gen import hgen  # noqa: E402
from paper_2008_12441_b200 import hmat as hm  # noqa: E402


def shard_time(cfg, P, g, warm=40, reps=20):
    dd = hm._dist(nranks=P, rank=g, device=0, external_exchange=True) if P > 1 else None
    h = hm.hmat_create_uninit(cfg.L, cfg.d, cfg.b, cfg.r, dd)
    try:
        r0, r1 = hm.hmat_local_rows(h)
        hgen.dev_fill_operator(cfg, lambda kind, level: hm.hmat_panel(h, kind, level), r0, r1, 0)
        n = r1 - r0
        x = torch.empty(cfg.nrhs, n, dtype=torch.float64, device="cuda")
        hgen.dev_fill_x(cfg, cfg.nrhs, 0, r0, r1, x.data_ptr(), n, 0)
        y = torch.empty_like(x)
        cnt = hm.hmat_exchange_size(h, cfg.nrhs) if P > 1 else 0
        xbuf = torch.zeros(max(1, cnt), dtype=torch.float64, device="cuda")

        def step():
            if P > 1:
                hm.hmat_project(h, x.t(), xbuf, cfg.nrhs)
                hm.hmat_expand(h, x.t(), xbuf, y.t(), cfg.nrhs)
            else:
                hm.hmat_matvec(h, x.t(), y.t(), cfg.nrhs)
        for _ in range(warm):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        return {"config": cfg.name, "P": P, "rank": g, "rows": [r0, r1], "ms_per_product": ms,
                "exchange_bytes": 8 * cnt, "factor_GB": cfg.factor_bytes / P / 1e9,
                "GBps": (cfg.factor_bytes / P + 16 * n * cfg.nrhs) / ms / 1e6}
    finally:
        hm.hmat_destroy(h)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    args = sys.argv[1:]
    name = args[0] if args and not args[0].isdigit() else "c4"
    Ps = [int(a) for a in args if a.isdigit()] or [1, 2, 4, 8]
    cfg = {**hgen.CONFIGS, **hgen.EXTRA_CONFIGS}[name]
    torch.cuda.set_device(0)
    for P in Ps:
        for g in sorted({0, P - 1}):
            print(json.dumps(shard_time(cfg, P, g)), flush=True)
