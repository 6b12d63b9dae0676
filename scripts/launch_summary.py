"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: launches, mean time and
share of the listed time per kernel (cold-cache serialised launches: compare shares, not absolutes).

    python scripts/launch_summary.py launches.csv [header line ...]
"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
tot = defaultdict(float)
cnt = defaultdict(int)
unit_scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}
for r in rows:
    name = r[4].split("(")[0].replace("void ", "")[:70]
    v = float(r[-1].replace(",", "")) * unit_scale.get(r[-2], 1e-3)
    tot[name] += v
    cnt[name] += 1
all_us = sum(tot.values())
for line in sys.argv[2:]:
    print(f"# {line}")
print(f"{'kernel':72s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:72s} {cnt[k]:8d} {tot[k] / cnt[k]:10.2f} {tot[k] / all_us * 100:6.1f}%")
