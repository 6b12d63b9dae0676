#!/bin/bash
# Same-box A/B of the fused detection + compaction and the balanced detection grid.
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_spmm.py -m gpu -q -x -p no:cacheprovider > $OUT/fuse_tests.txt 2>&1
echo "tests rc=$?"; tail -3 $OUT/fuse_tests.txt
for v in "PIT_DETECT_FUSE=0 PIT_DETECT_BALANCE=0" "PIT_DETECT_FUSE=0 PIT_DETECT_BALANCE=1" "PIT_DETECT_FUSE=1 PIT_DETECT_BALANCE=1" "PIT_DETECT_FUSE=0 PIT_DETECT_BALANCE=0" "PIT_DETECT_FUSE=1 PIT_DETECT_BALANCE=1"; do
  env $v timeout 300 python scripts/detect_fuse_probe.py 2>&1 | grep -v Warn
done
for v in "PIT_DETECT_FUSE=0 PIT_DETECT_BALANCE=0" "PIT_DETECT_FUSE=1 PIT_DETECT_BALANCE=1"; do
  env $v timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-moe --no-attn --no-opt --no-sweep --no-bert --no-c1 > $OUT/fuse_bench.json 2>/dev/null
  python -c "
import json; d=json.load(open('$OUT/fuse_bench.json')); print('$v', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], 'detect', d['detection']['ms'], d['detection']['frac'], 'idx', d['index_build']['ms'], d['index_build']['frac'], d['gpu_launches'])"
done
