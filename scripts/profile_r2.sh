#!/bin/bash
# Round-2 evidence: full bench line, launch list of the headline step, one `ncu --set full` capture per
# tcgen05 / detection kernel on the bench path (summaries go to profiles/r2/ by hand).
#   scripts/profile_r2.sh [names...]   (default: all)
OUT=gpurun_out; mkdir -p $OUT
NB="--no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-opt --no-sweep --no-bert --no-c1"
want() { [ -z "$ARGS" ] || [[ " $ARGS " == *" $1 "* ]]; }
ARGS="$*"
cap() {  # name kernel-regex skip command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $OUT/prof_$name -f \
    "$@" > $OUT/ncu_$name.log 2>&1
  python scripts/ncu_summary.py $OUT/prof_$name.ncu-rep 12 > $OUT/ncu_full_$name.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f $OUT/prof_$name.ncu-rep  # gpurun copies back at most 64 MiB
  echo "== $name"; grep -E "Kernel Name|gpu__time|utchmma.*pct|hmma_cycles|dram__bytes|lts__throughput" $OUT/ncu_full_$name.txt
}
if [ -z "$ARGS" ] || want bench; then
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
  timeout 1200 python bench.py > $OUT/r2_bench_full.json 2> $OUT/r2_bench_full.err; echo "bench rc=$?"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c1.csv \
    python bench.py --steps 2 --warmup 3 $NB > /dev/null 2>&1
  python scripts/launch_summary.py $OUT/launches_c1.csv > $OUT/launches_c1_summary.txt; cat $OUT/launches_c1_summary.txt
fi
want gk32 $ARGS && cap gk32 spmm_gk_kernel 3 python bench.py --workload pitk_c1_8192 --steps 1 --warmup 3 $NB
want detect $ARGS && cap detect detect 3 python bench.py --workload pitk_c1_8192 --steps 1 --warmup 3 $NB
want gk2 $ARGS && cap gk2 spmm_gk2 3 python bench.py --workload pitk_256_8192 --steps 1 --warmup 3 $NB
want gm32 $ARGS && cap gm32 rowgemm2 3 python bench.py --workload pitm_32_8192 --steps 1 --warmup 3 $NB
want bert $ARGS && cap bert_rg2 rowgemm2 2 python scripts/bert_probe.py --ncu
want moe $ARGS && cap moe_rg2t rowgemm2t 1 python scripts/rowgemm_probe.py --ncu
want attn $ARGS && cap attn_gk spmm_gk_kernel 2 python scripts/attn_warm.py
want sddmm $ARGS && cap sddmm_c3 sddmm_kernel 2 python scripts/sddmm_probe.py
want c4 $ARGS && cap c4_k3s_product rowgemm2t 1 python scripts/c4_probe.py 0.99 --ncu
want cols $ARGS && cap detect_cols detect_cols_slab 2 python scripts/dh_probe.py


ls $OUT/ncu_full_*.txt
