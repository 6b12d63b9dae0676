"""Top SASS instructions by warp-stall samples and by executed count from an ncu source page CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
k, e = idx["Warp Stall Sampling (All Samples)"], idx["Instructions Executed"]
data = [r for r in rows[2:] if len(r) > e]
tot = sum(float(r[k] or 0) for r in data)
tex = sum(float(r[e] or 0) for r in data)
print(f"total stall samples {tot:.0f}, executed warp instructions {tex:.0f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("--- by stall samples")
for r in sorted(data, key=lambda r: -float(r[k] or 0))[:n]:
    print(f"{r[k]:>7} {r[e]:>9} {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:100]}")
print("--- by executed")
for r in sorted(data, key=lambda r: -float(r[e] or 0))[:n]:
    print(f"{r[k]:>7} {r[e]:>9} {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:100]}")
