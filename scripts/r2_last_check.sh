#!/bin/bash
# End-of-round evidence on the final kernels: -m gpu suite, smoke, default bench line, launch list of
# the headline step, and the 2-rank expert-parallel rehearsal on one GPU (gloo plumbing).
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/last_gpu_tests.txt 2>&1
echo "pytest rc=$?"; tail -3 $OUT/last_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/last_smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 $OUT/last_smoke.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/last_smi.txt
timeout 1200 python bench.py > $OUT/last_bench.json 2> $OUT/last_bench.err; echo "bench rc=$?"; tail -c 300 $OUT/last_bench.json
NB="--no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-opt --no-sweep --no-bert --no-c1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/last_launches_c1.csv \
  python bench.py --steps 2 --warmup 3 $NB > /dev/null 2>&1
python scripts/launch_summary.py $OUT/last_launches_c1.csv > $OUT/last_launches_c1_summary.txt; head -8 $OUT/last_launches_c1_summary.txt
PIT_BENCH_PG=gloo PIT_BENCH_DEVICE=0 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
  --no-index-bench --no-attn --no-opt --no-sweep --no-bert --no-c1 > $OUT/last_rehearsal_ep2.json 2> $OUT/last_rehearsal_ep2.err
echo "rehearsal rc=$?"; tail -c 400 $OUT/last_rehearsal_ep2.json
