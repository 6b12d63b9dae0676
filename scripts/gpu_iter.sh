#!/bin/bash
# One GPU round-trip for kernel iteration: parity tests for the SpMM kernels, then per-workload
# kernel timings (no e2e / CPU baseline), optionally an ncu capture of one kernel.
#   scripts/gpu_iter.sh [pytest -k expr] [ncu kernel regex] [ncu workload]
set -u
K=${1:-spmm}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" -p no:cacheprovider > $OUT/iter_tests.txt 2>&1
tail -3 $OUT/iter_tests.txt
for w in pitk_c1_8192 pitk_128_8192 pitm_32_8192 bert_ffn1; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $( [ $w != pitk_c1_8192 ] && echo --no-index-bench --no-moe ) > $OUT/iter_$w.json 2>$OUT/iter_$w.err
  python - "$OUT/iter_$w.json" <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1]))
    r=d["roofline"]; det=d["detection"]
    ib=d.get('index_build',{}); print(f'idx16k={ib.get("ms")} ms {ib.get("achieved_GBps")} GB/s') if ib else None; mo=d.get('moe'); print('moe', mo) if mo else None; print(f'{d["config"]["name"]:14s} value={d["value"]:8.2f} TF/s  spmm={r["kernel_ms"]:.4f} ms ({r["achieved"]:.1f} TF/s, frac {r["frac"]:.3f})  detect={det["ms"]:.4f} ms ({det["achieved_GBps"]:.0f} GB/s) clocks={d["clocks"]["sm_mhz"]}')
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
if [ -n "${2:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o $OUT/prof_iter python bench.py --workload ${3:-pitk_c1_8192} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_iter.log 2>&1
  tail -2 $OUT/ncu_iter.log
fi
