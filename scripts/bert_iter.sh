#!/bin/bash
# C2 BERT iteration: probe timings (+ env variants), launch list of the eager step.
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/bert_probe.py > $OUT/bert_probe.txt 2>&1; cat $OUT/bert_probe.txt
for v in "PIT_SMALL_SINGLE=0"; do echo "== $v"; env $v timeout 300 python scripts/bert_probe.py 2>&1 | head -3 | tail -2; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/bert_launches.csv python scripts/bert_probe.py --ncu > /dev/null 2>&1
python scripts/launch_summary.py $OUT/bert_launches.csv 2>&1 | tail -20
