for v in 1 0; do
PIT_GK_RUNS=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed_op_tma.sum,l1tex__m_xbar2l1tex_read_bytes.sum --cache-control none --clock-control none -k regex:spmm_gk_kernel --csv python scripts/attn_warm.py 2>/dev/null | grep -E "spmm_gk" | tail -4 | awk -F'","' '{print "'runs=$v' " $(NF-2) " " $NF}'
done
