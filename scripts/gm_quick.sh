#!/bin/bash
# pitm_32_8192 + C4 (OPT FFN2) timings only
OUT=gpurun_out; mkdir -p $OUT
NB="--no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-sweep"
timeout 300 python bench.py --workload pitm_32_8192 --steps 10 --warmup 3 $NB > $OUT/gmq.json 2> $OUT/gmq.err
python - $OUT/gmq.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1])); r=d["roofline"]; o=d.get("opt_ffn2",{})
print("pitm_32_8192 value", d["value"], "spmm_ms", r["kernel_ms"], "TF", r["achieved"])
for z,v in o.get("by_zero_ratio",{}).items(): print("  opt", z, v["value"], "fwd", v["fwd_pit_m_TFLOPs"], "bwd", v["bwd_pit_k_TFLOPs"], "ms", v["ms_per_step"])
PY
