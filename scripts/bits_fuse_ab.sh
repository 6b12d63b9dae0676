#!/bin/bash
# Annotation-route index in one launch: parity tests, then same-box A/B of the C3 step parts.
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/bits_fuse_tests.txt 2>&1
echo "tests rc=$?"; tail -3 $OUT/bits_fuse_tests.txt
for v in 0 1 0 1; do echo "== PIT_BITS_FUSE=$v"; PIT_BITS_FUSE=$v timeout 300 python scripts/attn_parts.py 2>&1 | grep -v Warn; done
for v in 0 1; do
  PIT_BITS_FUSE=$v timeout 600 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-moe --no-opt --no-sweep --no-bert --no-c1 --no-index-bench > $OUT/bits_bench.json 2>/dev/null
  python -c "
import json; d=json.load(open('$OUT/bits_bench.json')); a=d['attention']; print('PIT_BITS_FUSE=$v', 'C1', d['value'], 'attn', a['value'], a['ms_per_step'], a['roofline']['frac'], {k: v['ms_per_step'] for k, v in a['variants'].items()})"
done
