#!/bin/bash
# C3 step launch list on the final kernels (annotation-route index in one launch).
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/attn_launches_final.csv python scripts/attn_parts.py > /dev/null 2>&1
python scripts/launch_summary.py $OUT/attn_launches_final.csv > $OUT/attn_launches_final_summary.txt; head -12 $OUT/attn_launches_final_summary.txt
