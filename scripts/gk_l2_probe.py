"""Is spmm_gk (32x1) latency-bound on first-touch DRAM misses? Time the kernel with the L2 flushed
before every call and with B (and A) left warm from the previous call, at N where B fits in L2
(2048: 32 MiB) and where it does not (8192: 128 MiB)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20 >> 2, dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
for N in (2048, 8192):
    w = dict(M=8192, K=8192, N=N, micro=(32, 1), axis="k", zero=0.9, tile=(32, 64, 32), name=f"probe{N}")
    A, B, live = bench.make_operands(w, seed=3, device=dev)
    plan = bench.make_plan(w)
    idx = pit.build_index_from_tensor(A, (32, 1), "k")
    C = pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx).array
    for mode in ("flushed", "warm"):
        ts = []
        for _ in range(10):
            if mode == "flushed":
                flush.zero_()
            else:
                pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx)
            e1.record(s)
            ts.append((e0, e1))
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in ts)
        print(f"N={N} {mode:8s} {ms:.4f} ms  {2.0 * N * live / ms / 1e9:.1f} TFLOP/s")
