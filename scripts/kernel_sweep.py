"""Per-kernel timing sweep over plan knobs (HMAT_* env vars) for one config.

    python scripts/kernel_sweep.py c4 "HMAT_STAGE_KB=36" "HMAT_STAGE_KB=24,HMAT_MAX_STAGES=8" ...

Builds the operator once per setting (device-generated seeded panels), runs
warm-up + timed matvecs with the library's event profiler, prints GB/s per kernel.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from gen import hgen  # noqa: E402
from paper_2008_12441_b200 import hmat as hm  # noqa: E402


def run(cfg, setting, reps=10):
    import dataclasses
    keys = []
    warm = 3
    for kv in filter(None, setting.split(",")):
        k, v = kv.split("=")
        if k == "NRHS":  # override the config's right-hand-side count
            cfg = dataclasses.replace(cfg, nrhs=int(v))
            continue
        if k == "REPS":  # timed matvecs
            reps = int(v)
            continue
        if k == "WARM":  # untimed matvecs first (e.g. enough to reach the sustained power cap)
            warm = int(v)
            continue
        os.environ[k] = v
        keys.append(k)
    try:
        h = (hm.hmat_create_standard_uninit if cfg.adm else hm.hmat_create_uninit)(cfg.L, cfg.d, cfg.b, cfg.r)
        info = hm.hmat_plan_query(cfg.L, cfg.d, cfg.b, cfg.r)
        r0, r1 = hm.hmat_local_rows(h)
        hgen.dev_fill_operator(cfg, lambda kind, level: hm.hmat_panel(h, kind, level), r0, r1, 0)
        n = r1 - r0
        x = torch.empty(cfg.nrhs, n, dtype=torch.float64, device="cuda")
        hgen.dev_fill_x(cfg, cfg.nrhs, 0, r0, r1, x.data_ptr(), n, 0)
        y = torch.empty_like(x)
        torch.cuda.synchronize()
        for _ in range(warm):
            hm.hmat_matvec(h, x.t(), y.t(), cfg.nrhs)
        hm.hmat_profile(h, True)
        hm.hmat_profile_read(h)
        for _ in range(reps):
            hm.hmat_matvec(h, x.t(), y.t(), cfg.nrhs)
        prof = hm.hmat_profile_read(h)
        hm.hmat_destroy(h)
        W, L, b, N = cfg.W, cfg.L - (1 if cfg.adm else 0), cfg.dcols, cfg.N
        pb = 8 * N * W * L + 8 * N * cfg.nrhs
        eb = 8 * N * (W * L + b) + 16 * N * cfg.nrhs
        pm = prof["project"][0] / reps  # per matvec (all passes)
        em = prof["expand"][0] / reps
        print(f"{cfg.name} [{setting or 'default'}] Rp={info.Rp} Re={info.Re} tpr={info.tpr} "
              f"ns_p={info.nstage_p} ns_e={info.nstage_e} grid={info.grid_p}/{info.grid_e} | "
              f"project {pm:.3f} ms {pb / pm / 1e6:.0f} GB/s | expand {em:.3f} ms {eb / em / 1e6:.0f} GB/s | "
              f"total {pm + em:.3f} ms ({2 * cfg.N * (2 * W * L + b) * cfg.nrhs / (pm + em) / 1e9:.2f} TFLOP/s) "
              f"launches/matvec={prof['project'][1] // reps}+{prof['expand'][1] // reps}", flush=True)
    finally:
        for k in keys:
            os.environ.pop(k, None)
        torch.cuda.empty_cache()


def parse_cfg(spec):
    """a BASELINE config name (c1..c5) or an ad-hoc shape 'd=3,L=4,b=64,r=32,nrhs=64'"""
    if spec in hgen.CONFIGS:
        return hgen.CONFIGS[spec]
    if spec in hgen.EXTRA_CONFIGS:
        return hgen.EXTRA_CONFIGS[spec]
    kv = dict(item.split("=") for item in spec.split(","))
    return hgen.HConfig(spec, **{k: int(v) for k, v in kv.items()}, seed=hgen.SEED_BASE + 99)


if __name__ == "__main__":
    cfg = parse_cfg(sys.argv[1])
    for setting in (sys.argv[2:] or [""]):
        run(cfg, setting)
