#!/bin/bash
# Final bench line after the config alignment, the reference arm, and the -m gpu suite + smoke.
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python bench.py > $OUT/final_bench.json 2> $OUT/final_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$OUT/final_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['config'], d['execution'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/final_ref.json 2> $OUT/final_ref.err; echo "ref rc=$?"; tail -c 300 $OUT/final_ref.json
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/final_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/final_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/final_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $OUT/final_smoke.txt
