"""Summarise an ncu --page source --csv dump: hottest SASS lines by stall samples.
usage: ncu -i rep --page source --csv --kernel-name regex:K | python scripts/ncu_hot.py [N]"""
import csv
import sys

rows = list(csv.reader(sys.stdin))
# first line is the kernel name row, second the header
start = 1 if rows and rows[0] and rows[0][0] == "Kernel Name" else 0
hdr = rows[start]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[start + 1:]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data if len(r) == len(hdr))
ins = sum(int(r[ix["Instructions Executed"]] or 0) for r in data if len(r) == len(hdr))
print(f"total samples {tot}, warp instructions {ins}")
top = sorted((r for r in data if len(r) == len(hdr)), key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:n]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in top:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    reasons = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:3]
    print(f"{100 * s / max(1, tot):5.1f}% {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} "
          f"exec={r[ix['Instructions Executed']]:>9} " + " ".join(f"{h}:{v}" for v, h in reasons if v))
