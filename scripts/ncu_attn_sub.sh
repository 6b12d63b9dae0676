NB="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-index-bench --no-moe --no-opt --no-sweep --no-bert --no-c1"
for v in 1 0; do
PIT_GM_SUB=$v timeout 600 ncu --set full --clock-control none -k regex:rowgemm_kernel -s 0 -c 1 -o gpurun_out/prof_attn_gm_sub$v -f python bench.py $NB > gpurun_out/ncu_attn_$v.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_attn_gm_sub$v.ncu-rep | grep -E "gpu__time|dram__bytes|lts__t_bytes|utchmma.*pct|xbar|tma|issue"
done
