#!/bin/bash
# pit:m contiguous-tile A/B: parity tests, then the pitm_32_8192 workload and the C4 section with
# PIT_GM_CONTIG unset (default 50%) and =0 (union-row tiles), same box.
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gm_tests.txt 2>&1
tail -3 $OUT/gm_tests.txt
NB="--no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-sweep"
for v in 50 0; do
  PIT_GM_CONTIG=$v timeout 300 python bench.py --workload pitm_32_8192 --steps 10 --warmup 3 $NB > $OUT/gm_$v.json 2> $OUT/gm_$v.err
  python - $OUT/gm_$v.json $v <<'PY'
import json,sys
d=json.load(open(sys.argv[1])); r=d["roofline"]; o=d.get("opt_ffn2",{})
print("contig", sys.argv[2], "pitm_32_8192 value", d["value"], "spmm_ms", r["kernel_ms"], "TF", r["achieved"])
for z,v in o.get("by_zero_ratio",{}).items(): print("  opt", z, v["value"], "fwd", v["fwd_pit_m_TFLOPs"], "bwd", v["bwd_pit_k_TFLOPs"], "ms", v["ms_per_step"], "err", v["max_rel_err_vs_f64"])
PY
done
