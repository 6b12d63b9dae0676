timeout 900 compute-sanitizer --tool racecheck --target-processes all python scripts/race_kernels.py > gpurun_out/r2_racecheck_kernels.txt 2>&1
echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|race_kernels done|Error" gpurun_out/r2_racecheck_kernels.txt | head -5
timeout 900 compute-sanitizer --tool memcheck python scripts/race_kernels.py > gpurun_out/r2_memcheck_kernels.txt 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|race_kernels done" gpurun_out/r2_memcheck_kernels.txt | head -3
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "moe or gk2 or dense or rowuniform or pitm_sparse or fullsize" 2>&1 | tail -2
