#!/bin/bash
# kernel timings of one workload under env knob sets: GK_W=workload GK_CFGS="A=1,B=2 C=3" scripts/gk_knobs.sh
OUT=gpurun_out; mkdir -p $OUT
W=${GK_W:-pitk_c1_8192}
for cfg in ${GK_CFGS:-"X=0"}; do
  cfg=${cfg//,/ }
  env $cfg timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-opt --no-sweep > $OUT/knob.json 2>$OUT/knob.err
  python -c "
import json,sys
d=json.load(open('$OUT/knob.json')); r=d['roofline']
print('$W $cfg', 'value', d['value'], 'kernel_ms', r['kernel_ms'], 'TF', r['achieved'], 'frac', r['frac'], 'clk', d['clocks']['sm_mhz'])" || tail -5 $OUT/knob.err
done
