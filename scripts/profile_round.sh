#!/bin/bash
# One GPU call that produces the round's evidence: full bench line, launch list, ncu --set full
# captures of the top kernels (summaries land in gpurun_out/, copied to profiles/<round>/ by hand).
OUT=gpurun_out; mkdir -p $OUT
NB="--no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-opt --no-sweep"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 900 python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c1.csv \
  python bench.py --steps 2 --warmup 3 $NB > /dev/null 2>&1
cap() {  # name regex workload
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o $OUT/prof_$1 \
    python bench.py --workload $3 --steps 1 --warmup 3 $NB > $OUT/ncu_$1.log 2>&1
}
cap gk32 spmm_gk_kernel pitk_c1_8192
cap gk128 spmm_gk_kernel pitk_128_8192
cap gk2 spmm_gk2 pitk_256_8192
cap detect detect pitk_c1_8192
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rowgemm2 -s 0 -c 1 -o $OUT/prof_rowgemm2 \
  python scripts/rowgemm_probe.py --ncu > $OUT/ncu_rowgemm.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_moe.csv python scripts/rowgemm_probe.py --ncu > /dev/null 2>&1
ls -la $OUT/*.ncu-rep
