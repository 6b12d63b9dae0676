#!/bin/bash
# One ncu --set full capture: NAME REGEX WORKLOAD [extra bench args]
OUT=gpurun_out; mkdir -p $OUT
NB="--no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-opt --no-sweep --no-bert"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o $OUT/prof_$1 -f \
  python bench.py --workload $3 --steps 1 --warmup 3 $NB ${@:4} > $OUT/ncu_$1.log 2>&1
tail -2 $OUT/ncu_$1.log
