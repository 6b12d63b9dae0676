#!/bin/bash
# C3 iteration: attention parity tests, then the bench attention section (variants) with env A/B knobs.
OUT=gpurun_out; mkdir -p $OUT
NB="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-opt --no-sweep --no-bert --no-c1"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "attn or attention or batched or masked or pitm" 2>&1 | tail -3
for v in ${VARIANTS:-PIT_X=0}; do
  env $v timeout 600 python bench.py $NB > $OUT/attn_$v.json 2>$OUT/attn_$v.err
  python - "$OUT/attn_$v.json" "$v" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))["attention"]
print(sys.argv[2], "best", d.get("plan"), d.get("ms_per_step"), "roofline", d.get("roofline", {}).get("frac"))
for k, v in d.get("variants", {}).items():
    print("   ", k, v["ms_per_step"], v["value"], v["graph_replay_equals_eager"], f'{v["max_rel_err_head0_vs_f64"]:.2e}')
PY
done
