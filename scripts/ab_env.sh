#!/bin/bash
# Same-box A/B of environment knobs on one workload: ab_env.sh WORKLOAD "ENV1" "ENV2" ...
# (each ENV a space-separated list of VAR=value, "-" for none)
OUT=gpurun_out; mkdir -p $OUT
W=$1; shift
NB="--no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-sweep --no-bert --no-opt"
for rep in 1 2; do
for e in "$@"; do
  envs=""; [ "$e" != "-" ] && envs="$e"
  env $envs timeout 300 python bench.py --workload $W --steps 20 --warmup 5 $NB > $OUT/abe.json 2>$OUT/abe.err
  python - $OUT/abe.json "$e" <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1])); r=d["roofline"]
    print(f'{sys.argv[2]:28s} {d["config"]["name"]:14s} step={d["value"]:8.2f} kernel={r["kernel_ms"]:.4f} ms {r["achieved"]:.1f} TF/s feed={(r.get("operand_feed") or {}).get("achieved_GBps")}')
except Exception as ex: print(sys.argv[2], "FAILED", ex, open(sys.argv[1].replace('.json','.err')).read()[-300:])
PY
done
done
