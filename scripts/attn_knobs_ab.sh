#!/bin/bash
# C3 P.V step under the gathered-K runtime knobs (same box), final kernels.
for v in "X=0" "PIT_GK_KS=64" "PIT_GK_SPLIT_FIRST=0" "PIT_GK_RUNS=0" "PIT_GK_SPLIT=0" "PIT_GK_NT=128" "X=0" "PIT_GK_KS=64"; do
  echo "== $v $(env $v timeout 300 python scripts/attn_parts.py 2>&1 | grep 'whole step')"
done
