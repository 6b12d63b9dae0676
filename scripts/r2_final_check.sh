#!/bin/bash
# Whole -m gpu suite + smoke + the tmem_alloc2 racecheck reproducer (built here).
OUT=gpurun_out; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/r2_gpu_tests.txt 2>&1
echo "pytest rc=$?"; tail -6 $OUT/r2_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2_smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 $OUT/r2_smoke.txt
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/tmem_alloc2_race scripts/probe/tmem_alloc2_race.cu > /dev/null 2>&1
for m in 0 1 2 3; do
  timeout 120 compute-sanitizer --tool racecheck /tmp/tmem_alloc2_race $m > $OUT/r2_race_probe_$m.txt 2>&1
  echo "race mode $m: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $OUT/r2_race_probe_$m.txt | tail -1)"
done
