timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_gk_kernel -s 2 -c 1 -o /tmp/prof_attn_gk -f python scripts/attn_warm.py > /dev/null 2>&1
ncu -i /tmp/prof_attn_gk.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null > /tmp/src.csv
python - <<'PY'
import csv
rows = list(csv.reader(open("/tmp/src.csv")))
# find header
hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
h = rows[hi]; data = rows[hi + 1:]
si = h.index("Warp Stall Sampling (All Samples)")
src_i = h.index("Source")
def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
tot = sum(f(r[si]) for r in data if len(r) > si) or 1.0
top = sorted((r for r in data if len(r) > si), key=lambda r: -f(r[si]))[:30]
for r in top:
    print(f"{f(r[si]) / tot * 100:5.1f}%  {r[0][:40]:40s} {r[src_i][:100]}")
PY
