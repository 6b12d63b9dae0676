#!/bin/bash
# Same-box A/B of the row-vector detection scan variants (rows in flight, L2 prefetch hint).
for v in 0 1 2 3 0 1 2 3; do
  PIT_DETECT_VARIANT=$v timeout 300 python scripts/detect_fuse_probe.py 2>&1 | grep "(32,1)" | sed "s/^/V=$v /"
done
timeout 600 python -m pytest tests/test_gpu_index.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
PIT_DETECT_VARIANT=3 timeout 600 python -m pytest tests/test_gpu_index.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
