#!/bin/bash
# needs a diagnostic build: PIT_DIAG=1 python -m paper_2301_10936_b200._build --force
OUT=gpurun_out; mkdir -p $OUT
for cfg in ${GK2_CFGS:-"PIT_GK_KS=128" "PIT_GK_KS=128 PIT_GK2_DIAG=1" "PIT_GK_KS=128 PIT_GK2_DIAG=2" "PIT_GK_KS=128 PIT_GK2_DIAG=3"}; do
  cfg=${cfg//,/ }
  env $cfg timeout 300 python bench.py --workload pitk_256_8192 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-opt --no-sweep > $OUT/gk2.json 2>$OUT/gk2.err
  python -c "
import json,sys
d=json.load(open('$OUT/gk2.json')); r=d['roofline']
print('$cfg', r['kernel_ms'], r['achieved'], r['operand_feed']['achieved_GBps'])" || tail -5 $OUT/gk2.err
done
