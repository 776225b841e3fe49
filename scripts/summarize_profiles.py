"""Turn gpurun_out/ ncu outputs into the committed profiles/ summaries.
usage: python scripts/summarize_profiles.py ROUND   (e.g. r01)"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(P, exist_ok=True)


def read_ncu_csv(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    return list(csv.DictReader(io.StringIO("".join(lines))))


# 1. launch list of the bench command: per-kernel count, total and share
rows = read_ncu_csv(os.path.join(G, "launches_c4.csv"))
agg = {}
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    t = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)  # -> us
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t
with open(os.path.join(P, f"{rnd}_launches_c4_summary.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none, command: "
            "python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e (c4)\n"
            "cold-cache, serialised launches: compare shares, not absolutes\n\n")
    hot = {k: v for k, v in agg.items() if "project" in k or "expand" in k}
    tot_hot = sum(v[1] for v in hot.values())
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = f"{100 * t / tot_hot:5.1f}% of matvec kernels" if k in hot else "setup (input generation)"
        f.write(f"{k:60s} launches={n:4d} total={t / 1e3:10.3f} ms mean={t / n / 1e3:9.3f} ms  {share}\n")
subprocess.run(["cp", os.path.join(G, "launches_c4.csv"), os.path.join(P, f"{rnd}_launches_c4.csv")])

# 2. dram traffic per launch of the c4 kernels (bench reads profiles/ncu_traffic.json)
rows = read_ncu_csv(os.path.join(G, "traffic_c4.csv"))
tr = {}
for r in rows:
    name = "project" if "project" in r["Kernel Name"] else "expand"
    d = tr.setdefault(name, {})
    d[r["Metric Name"]] = float(r["Metric Value"])
path = os.path.join(P, "ncu_traffic.json")
out = json.load(open(path)) if os.path.exists(path) else {}  # keep the other configs' entries
out["c4"] = {}
for k, d in tr.items():
    out["c4"][k] = {"dram_bytes_per_launch": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
                    "dram_bytes_read": d["dram__bytes_read.sum"], "dram_bytes_write": d["dram__bytes_write.sum"],
                    "ncu_duration_ns": d["gpu__time_duration.sum"],
                    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (one launch), {rnd}"}
with open(path, "w") as f:
    json.dump(out, f, indent=1)

# 3. key metrics of the full capture (c2)
rep = os.path.join(G, "prof_c2_full.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
            "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size"]
    with open(os.path.join(P, f"{rnd}_ncu_full_c2_summary.txt"), "w") as f:
        f.write(f"ncu --set full --clock-control none --import-source on, python scripts/kernel_sweep.py c2 ({rnd})\n\n")
        for r in rows[2:]:
            f.write(r[hdr.index("Kernel Name")] + "\n")
            for k in keys:
                if k in hdr:
                    f.write(f"  {k:60s} {r[hdr.index(k)]} {rows[1][hdr.index(k)]}\n")
            st = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled")
                  and not h.endswith("not_issued") and r[i] not in ("", "n/a")]
            tot = sum(float(v) for _, v in st) or 1.0
            f.write("  stall reasons (pc sampling):\n")
            for h, v in sorted(st, key=lambda t: -float(t[1]))[:6]:
                f.write(f"    {h[len('smsp__pcsamp_warps_issue_stalled_'):]:30s} {100 * float(v) / tot:5.1f}%\n")
            f.write("\n")
# 4. full captures of the bench's workload (c4) and of the DMMA kernels (c5): summaries,
#    reports, and their per-launch DRAM traffic (replaces step 2's entry for c4)
for cfg, what in (("c5", "python scripts/kernel_sweep.py c5 (full c5: N=2^21, W=224, 64 rhs)"),
                  ("c4", "python scripts/kernel_sweep.py c4 (full c4: N=2^24, W=48, 1 rhs; the bench's workload)")):
    rep = os.path.join(G, f"prof_{cfg}_full.ncu-rep")
    if os.path.exists(rep):
        subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "summarize_ncu.py"), rep,
                        os.path.join(P, f"{rnd}_ncu_full_{cfg}_summary.txt"), f"{what}, {rnd}", "--traffic", cfg],
                       check=True, capture_output=True)
        subprocess.run(["cp", rep, os.path.join(P, f"{rnd}_prof_{cfg}_full.ncu-rep")], check=True)
print("ok")
