timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none --clock-control none --csv --log-file gpurun_out/moe_warm.csv python scripts/moe_probe.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/moe_warm.csv")) if len(r) > 10]
seq=[]
for r in rows[1:]:
    if "pit::" not in r[4]: continue
    if r[-3]=="gpu__time_duration.sum": seq.append([r[4].split("(")[0][-40:], float(r[-1].replace(",",""))/1e3, 0])
    if r[-3]=="dram__bytes_read.sum" and seq: seq[-1][2]=float(r[-1].replace(",",""))/1e6
for name,t,b in seq[-7:]:
    print(f"{name:42s} {t:8.1f} us  dram {b:8.1f} MB")
PY
