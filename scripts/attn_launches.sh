#!/bin/bash
# C3 step breakdown (graph parts) and the ncu launch list of the step's kernels.
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/attn_parts.py 2>&1 | grep -v Warn
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/attn_launches.csv python scripts/attn_parts.py > /dev/null 2>&1
python scripts/launch_summary.py $OUT/attn_launches.csv 2>&1 | head -20
