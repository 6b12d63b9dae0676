"""Summarise an ncu report: headline throughput metrics + top stall sites (for profiles/)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u = r[0], r[1]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]
for row in r[2:]:
    for name in want:
        if name in h:
            i = h.index(name)
            print(f"{name:75s} {row[i]:>20s} {u[i]}")
    print()
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    s = list(csv.reader(src.splitlines()))
    hh = s[1]; rows = s[2:]
    si = hh.index("Warp Stall Sampling (All Samples)"); sc = hh.index("Source")
    tot = sum(float(x[si] or 0) for x in rows)
    for x in sorted(rows, key=lambda x: -float(x[si] or 0))[:int(sys.argv[2])]:
        print(f"{float(x[si]) / tot * 100:5.1f}%  {x[0][-5:]}  {x[sc][:100]}")
