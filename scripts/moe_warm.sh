timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none --clock-control none --csv --log-file gpurun_out/moe_warm.csv python scripts/moe_probe.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/moe_warm.csv")) if len(r) > 10]
t=collections.defaultdict(list); b=collections.defaultdict(list)
for r in rows[1:]:
    name=r[4].split("(")[0][-45:]
    if r[-3]=="gpu__time_duration.sum": t[name].append(float(r[-1].replace(",","")))
    if r[-3]=="dram__bytes_read.sum": b[name].append(float(r[-1].replace(",","")))
for k in t:
    print(f"{k:46s} n={len(t[k]):3d} last={t[k][-1]/1e3:8.1f} us  dram_read={b[k][-1]/1e6 if b[k] else 0:8.1f} MB")
PY
