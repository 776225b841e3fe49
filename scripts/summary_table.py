"""Rebuild the table of profiles/<round>_summary.md from profiles/<round>_bench_*.json.
usage: python scripts/summary_table.py r01"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = []
for c in ["c1", "c2", "c3", "c4", "c5", "s2", "c2strict", "c2r2", "c2r4", "c2r8", "c2r16", "c4r2", "c4r4", "c4r8", "c4r16", "s2r16",
          "c4_long", "c4r8_long", "c4r16_long", "c5_long"]:
    p = os.path.join(ROOT, "profiles", f"{rnd}_bench_{c}.json")
    if not os.path.exists(p):
        continue
    d = json.load(open(p))
    r, ph, e, clk, cpu = d["roofline"], d["phase_ms_per_step"], d["e2e"], d["clocks"], d["cpu_baseline"]
    # energy only over >= 2 s of timed steps: nvidia-smi's power.draw is a 1-s average
    long_run = clk.get("j_per_matvec") and d["ms_per_step"] * d["steps"] >= 2000.0
    rs = r.get("frac_of_read_stream")
    e2e = f"{e['value']:,.1f} / {e['blocking']['value']:,.1f}" if e else "—"  # (--no-e2e runs: none)
    rows.append(f"| {c} | {d['value']:,.1f} | {d['ms_per_step']:.3f} | {r['bound']} | {r['kernel']} | "
                f"{r['achieved']:,.1f} {r['unit']} | {r['peak']:,.1f} | {r['frac']:.3f} | "
                f"{'%.3f' % rs if rs else '—'} | {ph['project']:.3f} | {ph['expand']:.3f} | "
                f"{e2e} | "
                f"{'%.4g' % cpu['value'] if cpu else '—'} | "
                f"{clk['sm_mhz']:.0f}, {', '.join(clk['reasons']) or '-'} | "
                f"{'%.0f W, %.1f J' % (clk['power_w'], clk['j_per_matvec']) if long_run else '—'} |")
hdr = ("| cfg | matvec/s | ms/step | bound | dominant kernel | achieved | peak | frac | frac of 7.3 TB/s read stream "
       "| project ms | expand ms | e2e streaming / blocking (matvec/s) | CPU oracle (matvec/s, all cores) | SM MHz, throttle "
       "| board power, energy per matvec |\n"
       "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
print(hdr)
print("\n".join(rows))
