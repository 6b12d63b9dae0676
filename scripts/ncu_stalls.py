"""Per-instruction stall breakdown from an ncu report's source page (SASS view).

    python scripts/ncu_stalls.py report.ncu-rep [top_n] [addr_lo addr_hi]
"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
body = rows[2:]
ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
if len(sys.argv) > 4:
    lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
    body = [r for r in body if lo <= int(r[ia][-5:], 16) <= hi]
tot = sum(float(r[iall] or 0) for r in body)
agg = Counter()
for r in body:
    for i in stall_cols:
        agg[h[i]] += float(r[i] or 0)
print("total samples", tot)
print("  ".join(f"{k}={v / tot * 100:.1f}%" for k, v in agg.most_common(10)))
for r in sorted(body, key=lambda r: -float(r[iall] or 0))[:top]:
    reasons = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
    rs = " ".join(f"{n}:{v:.0f}" for v, n in reasons if v > 0)
    print(f"{float(r[iall]) / tot * 100:5.1f}% {r[ia][-5:]} ex={r[iex]:>8s} {r[isrc][:60]:60s} {rs}")
