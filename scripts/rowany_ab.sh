#!/bin/bash
# Same-box A/B: whole-row detection with 32- or 16-row blocks (C2's (1, 768) padding rows).
for v in 32 16 32 16; do
  PIT_ROWANY_RB=$v timeout 300 python scripts/detect_fuse_probe.py 2>&1 | grep BERT | sed "s/^/RB=$v /"
done
PIT_ROWANY_RB=16 timeout 600 python -m pytest tests/test_gpu_index.py tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider -k "whole_row or fuzz or repeats" 2>&1 | tail -1
