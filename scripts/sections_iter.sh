#!/bin/bash
# bench sections C2 + C4 only (quick look at the section JSON)
NB="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-sweep --no-c1"
timeout 900 python bench.py $NB > gpurun_out/sections.json 2> gpurun_out/sections.err; echo rc=$?
python - <<'PY'
import json
d = json.load(open("gpurun_out/sections.json"))
print(json.dumps(d.get("bert_ffn1"), indent=None)[:1500])
for k, v in d.get("opt_ffn2", {}).get("by_zero_ratio", {}).items():
    print(k, v)
PY
tail -3 gpurun_out/sections.err
