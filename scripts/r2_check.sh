#!/bin/bash
# Round-2 checkpoint: full -m gpu suite, smoke, default bench line.
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/r2_gpu_tests.txt 2>&1
echo "pytest rc=$?"; tail -15 $OUT/r2_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2_smoke.txt 2>&1; echo "smoke rc=$?"; tail -3 $OUT/r2_smoke.txt
timeout 900 python bench.py > $OUT/r2_bench.json 2> $OUT/r2_bench.err; echo "bench rc=$?"; tail -c 3000 $OUT/r2_bench.json
