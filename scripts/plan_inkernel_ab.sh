#!/bin/bash
# Split plan inside spmm_gk (first CTA computes it) vs the separate plan launch: suite + C3 A/B.
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/plan_tests.txt 2>&1
echo "tests rc=$?"; tail -2 $OUT/plan_tests.txt
for v in 0 1 0 1; do echo "== PIT_GK_PLAN_INKERNEL=$v $(PIT_GK_PLAN_INKERNEL=$v timeout 300 python scripts/attn_parts.py 2>&1 | grep -E 'whole|SpMM only' | tr '\n' ' ')"; done
for v in 0 1; do
  PIT_GK_PLAN_INKERNEL=$v timeout 600 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-moe --no-opt --no-sweep --no-bert --no-c1 --no-index-bench > $OUT/plan_bench.json 2>/dev/null
  python -c "
import json; d=json.load(open('$OUT/plan_bench.json')); a=d['attention']; print('PIT_GK_PLAN_INKERNEL=$v', 'attn', a['value'], a['ms_per_step'], a['roofline']['frac'], a['variants']['pit:k (128,1) column-major P'])"
done
