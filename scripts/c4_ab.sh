NB="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-attn --no-sweep --no-bert --no-c1"
for v in "PIT_GM_PART16=0" "PIT_GM_PART16=1"; do
  env $v timeout 600 python bench.py $NB > gpurun_out/c4ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/c4ab.json'))['opt_ffn2']['by_zero_ratio']['0.99']; print('$v', d['ms_per_step'], d['fwd_ms'], d['max_rel_err_vs_f64'])"
done
PIT_GM_PART16=1 timeout 300 python -m pytest tests/test_gpu_pitm_sparse.py -x -q -p no:cacheprovider 2>&1 | tail -2
