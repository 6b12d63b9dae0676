"""Summarise an ncu report: headline throughput metrics (tensor pipe, DRAM, L2, issue) per kernel and,
optionally, the top stall sites (for profiles/).

    python scripts/ncu_summary.py report.ncu-rep [n_stall_lines]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u = r[0], r[1]
# metric names as ncu prints them (some carry a section prefix such as "TPC.TriageCompute."): matched by suffix
want = ["Kernel Name", "launch__grid_size", "launch__cluster_dim_x", "gpu__time_duration.sum",
        # tcgen05 (UTC*MMA) bf16 work: executed FLOPs and their share of the tensor peak, subpipe busy
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread"]


def col(name):
    for i, c in enumerate(h):
        if c == name or c.endswith("." + name):
            return i
    return None


for row in r[2:]:
    for name in want:
        i = col(name)
        if i is not None:
            print(f"{name:90s} {row[i]:>24s} {u[i]}")
    print()
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    s = list(csv.reader(src.splitlines()))
    hh = s[1]
    rows = s[2:]
    si = hh.index("Warp Stall Sampling (All Samples)")
    sc = hh.index("Source")
    tot = sum(float(x[si] or 0) for x in rows) or 1.0
    for x in sorted(rows, key=lambda x: -float(x[si] or 0))[:int(sys.argv[2])]:
        print(f"{float(x[si]) / tot * 100:5.1f}%  {x[0][-5:]}  {x[sc][:100]}")
