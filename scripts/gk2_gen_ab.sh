#!/bin/bash
# spmm_gk2 producer-rotation A/B (generic arrays vs hand-rotated, build_alt/libpit_gk2hand.so) on
# the 256x1 and 128x1 @ 90% workloads, alternating, twice.
OUT=gpurun_out; mkdir -p $OUT
NB="--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-opt --no-sweep --no-bert --no-c1"
for rep in 1 2; do
  for lib in "" build_alt/libpit_gk2hand.so; do
    for wl in pitk_256_8192 pitk_128_8192; do
      PIT_LIB_PATH=$lib timeout 600 python bench.py --workload $wl $NB > $OUT/gk2ab.json 2>/dev/null
      python - "$OUT/gk2ab.json" "${lib:-default} $wl" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f'{sys.argv[2]:48s} step {d["value"]:.1f} TF/s kernel {d["roofline"]["achieved"]:.1f} ({d["roofline"]["kernel"]})')
PY
    done
  done
done
