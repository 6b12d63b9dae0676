"""C3 step broken into CUDA-graph parts (L2 flushed before each replay, mean of 50): the whole
step, the index build alone, the SpMM alone over a prebuilt index (split plan + spmm_gk)."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402

dev = torch.device("cuda", 0)
s = torch.cuda.current_stream()
flush = torch.empty(bench.FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
heads, seq, hd = 12, 4096, 64
blocks = bench.longformer_blocks(heads, seq, np.random.default_rng(3))
ann = pit.from_bits(blocks.reshape(heads * seq // 32, seq // 64), (heads * seq, seq), (32, 64)).on_device(dev)
P = torch.randn((heads, seq, seq), device=dev, dtype=torch.bfloat16)
V = torch.randn((heads, seq, hd), device=dev, dtype=torch.bfloat16)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
if reg.get("matmul", (128, 64, 256)) is None:
    reg.register(pit.TileKernelDescriptor("matmul", (128, 64, 256), "a"))
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=seq, k=seq, n=hd))
plan = pit.forced_plan(expr, "k", reg, tile_shape=(128, 64, 256))
Pk = pit.stack_slices(P, plan)
del P


def graphed(fn):
    side = torch.cuda.Stream()
    side.wait_stream(s)
    with torch.cuda.stream(side):
        for _ in range(2):
            fn()
    s.wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def timed(g, n=50):
    for _ in range(5):
        g.replay()
    ev = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.mean(p.elapsed_time(q) for p, q in ev) * 1e3


idx = pit.build_index(ann, (128, 1), "k")
print(f"whole step                {timed(graphed(lambda: pit.run_batched_matmul_with_index(plan, Pk, V, pit.build_index(ann, (128, 1), 'k')))):6.1f} us")
print(f"index build only          {timed(graphed(lambda: pit.build_index(ann, (128, 1), 'k'))):6.1f} us")
print(f"SpMM only (prebuilt idx)  {timed(graphed(lambda: pit.run_batched_matmul_with_index(plan, Pk, V, idx))):6.1f} us")
x = torch.zeros(256, device=dev)
print(f"one trivial kernel        {timed(graphed(lambda: x.add_(1))):6.1f} us")
