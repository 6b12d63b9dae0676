timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_gk_kernel -s 2 -c 1 -o gpurun_out/prof_attn_gk -f python scripts/attn_warm.py > gpurun_out/ncu_attn_gk.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_attn_gk.ncu-rep 14 > gpurun_out/ncu_full_attn_gk.txt 2>&1
ncu -i gpurun_out/prof_attn_gk.ncu-rep --page details --csv 2>/dev/null | grep -i "stall\|warp cycles per issued\|Eligible\|Active Warps\|Theoretical Occ" | head -30 > gpurun_out/ncu_attn_gk_details.txt
rm -f gpurun_out/prof_attn_gk.ncu-rep
cat gpurun_out/ncu_full_attn_gk.txt | tail -40
