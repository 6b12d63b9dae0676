#!/bin/bash
# Re-entry check after a container rebuild: whole -m gpu suite, default bench line, C2 probe.
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/reentry_gpu_tests.txt 2>&1
echo "pytest rc=$?"; tail -3 $OUT/reentry_gpu_tests.txt
timeout 900 python bench.py > $OUT/reentry_bench.json 2> $OUT/reentry_bench.err
echo "bench rc=$?"; tail -c 600 $OUT/reentry_bench.json
timeout 300 python scripts/bert_probe.py > $OUT/reentry_bert_probe.txt 2>&1; cat $OUT/reentry_bert_probe.txt | tail -30
