python scripts/c4_probe.py 0.99; PIT_GM_SPARSE=0 python scripts/c4_probe.py 0.99 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/c4_probe.py 0.99 --ncu > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/c4_launches.csv 2>/dev/null | grep "pit::"
timeout 300 python -m pytest tests/test_gpu_pitm_sparse.py tests/test_gpu_moe.py -x -q -p no:cacheprovider 2>&1 | grep -E "Error|error|assert|passed|failed" | head -20
python scripts/rowgemm_probe.py 2>&1 | tail -4
