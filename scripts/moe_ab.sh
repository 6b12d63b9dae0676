NB="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-attn --no-opt --no-sweep --no-bert --no-c1"
for v in ${VARIANTS:-PIT_MOE_PACK=0 PIT_MOE_PACK=1}; do
  env $v timeout 600 python bench.py $NB > gpurun_out/moe_ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/moe_ab.json'))['moe']; print('$v', d['ms_per_layer'], d['value'], d['roofline']['frac'])"
done
python scripts/rowgemm_probe.py | tail -1
