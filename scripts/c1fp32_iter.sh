python scripts/c1fp32_probe.py
timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/c1fp32.csv python scripts/c1fp32_probe.py --ncu > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/c1fp32.csv")) if len(r) > 10]
for r in rows[1:]:
    if "pit::" in r[4] and r[-3]=="gpu__time_duration.sum": print(r[4].split("(")[0][-50:], float(r[-1].replace(",",""))/1e3, "us")
PY
