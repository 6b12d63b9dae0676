#!/bin/bash
# index build at 16384^2 (K1 scan + compaction) for the in-tree and an alternative library
for L in "" ${ALT_LIB:-build_alt/lib_8ecdd07.so} "" ${ALT_LIB:-build_alt/lib_8ecdd07.so}; do
  PIT_LIB_PATH=$L timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-moe --no-attn --no-opt --no-sweep > gpurun_out/idx.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/idx.json')); i=d['index_build']; print('lib=$L', i['ms'], i['achieved_GBps'], i['frac'])"
done
