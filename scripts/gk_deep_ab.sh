#!/bin/bash
# spmm_gk slot-index lookahead A/B on one box: the default build vs build_alt/libpit_deep4.so
# (LIBS: alternative builds, e.g. PIT_GK_IDX_DEPTH=3/5/6 from scripts/build_alt.sh). Headline step + C3 attention, alternating, twice.
OUT=gpurun_out; mkdir -p $OUT
NB="--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-opt --no-sweep --no-bert --no-c1"
for rep in 1 2; do
  for lib in "" ${LIBS:-build_alt/libpit_deep4.so}; do
    PIT_LIB_PATH=$lib timeout 600 python bench.py $NB > $OUT/deep_$rep.json 2>/dev/null
    python - "$OUT/deep_$rep.json" "${lib:-default}" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
a = d["attention"]
print(f'{sys.argv[2]:32s} C1 {d["value"]:.1f} TF/s gk {d["roofline"]["achieved"]:.1f} kernel_ms {d["roofline"]["kernel_ms"]:.4f} | C3 {a["ms_per_step"]} frac {a["roofline"]["frac"]}')
PY
  done
done
