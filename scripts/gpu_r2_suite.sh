#!/bin/bash
# Round-2 GPU check: the whole -m gpu suite, then the tmem_alloc2 racecheck reproducer.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} > $OUT/r2_gpu_tests.txt 2>&1
echo "pytest rc=$?"; tail -5 $OUT/r2_gpu_tests.txt
if [ -x scripts/probe/tmem_alloc2_race ]; then
  for m in 0 1 2 3 4 5 6 7 8 9 10; do
    timeout 120 compute-sanitizer --tool racecheck scripts/probe/tmem_alloc2_race $m > $OUT/r2_race_probe_$m.txt 2>&1
    tail -3 $OUT/r2_race_probe_$m.txt
  done
fi
