#!/bin/bash
# split gathered-K units A/B: parity, then the C3 attention kernel alone with PIT_GK_SPLIT=1/0
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/split_tests.txt 2>&1
tail -3 $OUT/split_tests.txt
for v in 1 0; do
  PIT_GK_SPLIT=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/attn_k128.py 128 > $OUT/split_$v.csv 2>&1
  echo "split=$v"; grep micro $OUT/split_$v.csv; grep -h gpu__time $OUT/split_$v.csv | tail -4 | awk -F'","' '{print $5, $NF}' | cut -c1-60,200-
done
PIT_GK_SPLIT=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-sweep --no-opt > $OUT/split_bench.json 2>$OUT/split_bench.err
python -c "import json; d=json.load(open('$OUT/split_bench.json')); print(json.dumps(d['attention']['variants'])); print('value', d['value'])"
