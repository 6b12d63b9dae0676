timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/c4_warm.csv python scripts/c4_probe.py 0.99 --ncu > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/c4_warm.csv")) if len(r) > 10]
h=rows[0]
for r in rows[1:]:
    if "pit::" in r[4] and r[-3] in ("gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum"):
        print(r[4].split("(")[0][-50:], r[-3], r[-2], r[-1])
PY
