#!/bin/bash
# C4 iteration: high-sparsity pit:m tests, then the bench C4 section (both zero ratios), env A/B.
OUT=gpurun_out; mkdir -p $OUT
NB="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-sweep --no-bert --no-c1"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${PYTEST_K:-pitm_sparse or opt or masked or pitm}" 2>&1 | tail -4
for v in "PIT_GM_SPARSE=1" "PIT_GM_SPARSE=0"; do
  env $v timeout 600 python bench.py $NB > $OUT/opt_$v.json 2>$OUT/opt_$v.err
  python - "$OUT/opt_$v.json" "$v" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))["opt_ffn2"]
    for k, v in d["by_zero_ratio"].items():
        print(sys.argv[2], k, {x: v[x] for x in ("value", "ms_per_step", "fwd_pit_m_TFLOPs", "bwd_pit_k_TFLOPs", "max_rel_err_vs_f64", "graph_replay_equals_eager")})
except Exception as e:
    print(sys.argv[2], "FAILED", e, open(sys.argv[1].replace(".json", ".err")).read()[-1500:])
PY
done
