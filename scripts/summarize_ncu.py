"""Summarise one `ncu --set full` report (key metrics + top stall reasons per kernel)
and optionally record its per-launch DRAM traffic for bench.py's roofline.traffic.

    python scripts/summarize_ncu.py gpurun_out/prof_c5_full.ncu-rep profiles/r01_ncu_full_c5_summary.txt \
        "python scripts/kernel_sweep.py c5 (round 1)" [--traffic c5]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def main():
    rep, out, what = sys.argv[1], sys.argv[2], sys.argv[3]
    traffic_cfg = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    per_kernel = {}
    with open(out, "w") as f:
        f.write(f"ncu --set full --clock-control none --import-source on, {what}\n\n")
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            f.write(name + "\n")
            for k in KEYS:
                if k in hdr:
                    f.write(f"  {k:80s} {r[hdr.index(k)]} {units[hdr.index(k)]}\n")
            st = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled")
                  and not h.endswith("not_issued") and r[i] not in ("", "n/a")]
            tot = sum(float(v) for _, v in st) or 1.0
            f.write("  stall reasons (pc sampling):\n")
            for h, v in sorted(st, key=lambda t: -float(t[1]))[:6]:
                f.write(f"    {h[len('smsp__pcsamp_warps_issue_stalled_'):]:30s} {100 * float(v) / tot:5.1f}%\n")
            f.write("\n")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(r[hdr.index("dram__bytes_read.sum")]) * scale[units[hdr.index("dram__bytes_read.sum")]]
            wr = float(r[hdr.index("dram__bytes_write.sum")]) * scale[units[hdr.index("dram__bytes_write.sum")]]
            kind = "project" if "project" in name else "expand"
            per_kernel[kind] = {"dram_bytes_per_launch": rd + wr, "dram_bytes_read": rd, "dram_bytes_write": wr,
                                "source": f"ncu --set full (one launch): {what}"}
    if traffic_cfg:
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        data = json.load(open(path)) if os.path.exists(path) else {}
        data[traffic_cfg] = per_kernel
        with open(path, "w") as f:
            json.dump(data, f, indent=1)
    print(open(out).read())


if __name__ == "__main__":
    main()
