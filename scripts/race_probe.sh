nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/tmem_alloc2_race scripts/probe/tmem_alloc2_race.cu > /dev/null 2>&1
for m in 3 4 5 6 7 8 9 10; do
  timeout 120 compute-sanitizer --tool racecheck /tmp/tmem_alloc2_race $m > gpurun_out/r2_race_probe_$m.txt 2>&1
  echo "mode $m (variant $((m-3))): $(grep -E 'RACECHECK SUMMARY' gpurun_out/r2_race_probe_$m.txt | tail -1) $(grep -o 'Write access at [^ ]*' gpurun_out/r2_race_probe_$m.txt | head -1)"
done
