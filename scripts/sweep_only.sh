#!/bin/bash
# sparsity sweep + attention only (fast perf check)
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-opt > gpurun_out/sweep.json 2>gpurun_out/sweep.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/sweep.json"))
print("c1 value", d["value"], "spmm TF", d["roofline"]["achieved"])
for k,v in d["sparsity_sweep"]["by_microtile_and_zero_ratio"].items(): print(k, v["effective_TFLOPs"], v["spmm_ms"])
a=d["attention"]; print("attn", {k:(v["ms_per_step"],v["value"]) for k,v in a["variants"].items()})
PY
