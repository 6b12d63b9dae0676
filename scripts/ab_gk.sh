#!/bin/bash
# Same-box A/B of the gathered-K kernels: parity tests on the working tree, then the C1 headline and
# 128x1 workloads with the working-tree library and with build_alt/libpit_$ALT.so.
OUT=gpurun_out; mkdir -p $OUT
ALT=${ALT:-HEAD}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${PYTEST_K:-pit_k or golden or gk or batched or fullsize}" > $OUT/ab_tests.txt 2>&1
tail -2 $OUT/ab_tests.txt
NB="--no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-sweep --no-bert --no-opt"
for rep in 1 2; do
for lib in new alt; do
  for w in ${WORKLOADS:-pitk_c1_8192 pitk_128_8192}; do
    if [ $lib = alt ]; then export PIT_LIB_PATH=build_alt/libpit_$ALT.so; else unset PIT_LIB_PATH; fi
    timeout 300 python bench.py --workload $w --steps 20 --warmup 5 $NB > $OUT/ab_${lib}_$w.json 2>$OUT/ab_${lib}_$w.err
    python - $OUT/ab_${lib}_$w.json $lib <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1])); r=d["roofline"]
    print(f'{sys.argv[2]:4s} {d["config"]["name"]:14s} step={d["value"]:8.2f} TF/s kernel={r["kernel_ms"]:.4f} ms {r["achieved"]:.1f} TF/s feed={(r.get("operand_feed") or {}).get("achieved_GBps")} clk={d["clocks"]["sm_mhz"]}')
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
  done
done
done
unset PIT_LIB_PATH
