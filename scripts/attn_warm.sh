timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none --clock-control none --csv --log-file gpurun_out/attn_warm.csv python scripts/attn_warm.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/attn_warm.csv")) if len(r) > 10]
seen=collections.OrderedDict()
for r in rows[1:]:
    name=r[4].split("(")[0][-45:]
    if "pit::" not in r[4]: continue
    seen.setdefault(name, {})[r[-3]] = r[-1]
for k, v in seen.items():
    print(f"{k:46s} {float(v.get('gpu__time_duration.sum','0').replace(',',''))/1e3:8.1f} us  dram {float(v.get('dram__bytes_read.sum','0').replace(',',''))/1e6:8.1f} MB")
PY
