#!/bin/bash
# Round evidence (second pass of round 1): full bench line, launch lists of the C1 step and the C3
# attention step, ncu --set full captures of spmm_gk (C1), the split attention kernel and the
# masked pit:m rowgemm2 (CTA pairs), with summaries. Copy the summaries to profiles/r1/ by hand.
OUT=gpurun_out; mkdir -p $OUT
NB="--no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-opt --no-sweep"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 900 python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c1.csv \
  python bench.py --steps 2 --warmup 3 $NB > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_attn.csv \
  python scripts/attn_k128.py 128 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_gk_kernel -s 3 -c 1 -o $OUT/prof_gk32 \
  python bench.py --workload pitk_c1_8192 --steps 1 --warmup 3 $NB > $OUT/ncu_gk32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_gk_kernel -s 3 -c 1 -o $OUT/prof_attn_split \
  python scripts/attn_k128.py 128 > $OUT/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rowgemm2_kernel -s 2 -c 1 -o $OUT/prof_pitm_contig \
  python bench.py --workload pitm_32_8192 --steps 1 --warmup 3 $NB > $OUT/ncu_pitm.log 2>&1
for r in gk32 attn_split pitm_contig; do
  [ -f $OUT/prof_$r.ncu-rep ] && python scripts/ncu_summary.py $OUT/prof_$r.ncu-rep 12 > $OUT/ncu_full_$r.txt 2>&1
done
python scripts/launch_summary.py $OUT/launches_c1.csv "C1-8192 step (bench.py --steps 2 --warmup 3, graph capture + warm-up included)" > $OUT/launches_c1_summary.txt
python scripts/launch_summary.py $OUT/launches_attn.csv "C3 attention P.V, pit:k (128,1), split units (scripts/attn_k128.py 128; 11 steps)" > $OUT/launches_attn_summary.txt
ls -la $OUT/*.ncu-rep
