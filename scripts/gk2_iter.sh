#!/bin/bash
# CTA-pair gathered-K iteration: parity for every t0, then 256x1 / 128x1 timings under the knobs.
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_batched.py -m gpu -x -q -p no:cacheprovider > $OUT/gk2_tests.txt 2>&1
tail -3 $OUT/gk2_tests.txt
for cfg in "PIT_GK2=1 PIT_GK_KS=64" "PIT_GK2=1 PIT_GK_KS=128" "PIT_GK2=0"; do
  env $cfg timeout 300 python bench.py --workload pitk_256_8192 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-opt --no-sweep > $OUT/gk2.json 2>$OUT/gk2.err
  python -c "
import json,sys
d=json.load(open('$OUT/gk2.json')); r=d['roofline']
print('$cfg', d['value'], r['kernel'], r['kernel_ms'], r['achieved'], r['frac'], r['operand_feed'])" || tail -5 $OUT/gk2.err
done
