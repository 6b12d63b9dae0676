"""C3 attention step as a CUDA graph (index build from the block mask + split SpMM): replay output vs
the eager result, and the replay time (CUDA events, L2 flushed). PIT_PDL=0/1 A/B."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402

dev = torch.device("cuda", 0)
heads, seq, hd = 12, 4096, 64
blocks = bench.longformer_blocks(heads, seq, np.random.default_rng(3))
ann = pit.from_bits(blocks.reshape(heads * seq // 32, seq // 64), (heads * seq, seq), (32, 64)).on_device(dev)
g = torch.Generator(device=dev).manual_seed(5)
emask = torch.from_numpy(blocks).to(dev).repeat_interleave(32, 1).repeat_interleave(64, 2)
P = torch.randn((heads, seq, seq), device=dev, dtype=torch.bfloat16, generator=g) * emask.to(torch.bfloat16)
del emask
V = torch.randn((heads, seq, hd), device=dev, dtype=torch.bfloat16, generator=g)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=seq, k=seq, n=hd))
tile = (128, 64, 256)
if reg.get("matmul", tile) is None:
    reg.register(pit.TileKernelDescriptor("matmul", tile, "attn"))
plan = pit.forced_plan(expr, "k", reg, tile_shape=tile)
A3k = pit.stack_slices(P, plan)
ref = P.float() @ V.float()
del P


def step():
    return pit.run_batched_matmul_with_index(plan, A3k, V, pit.build_index(ann, (128, 1), "k"))


eager = step().float()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    for _ in range(2):
        step()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    out = step()
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
ts, errs = [], []
for i in range(10):
    out.zero_()
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    graph.replay()
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    errs.append(float((out.float() - ref).abs().max() / ref.abs().max()))
print(f"graph replay {statistics.median(ts):.4f} ms  max err vs fp32 {max(errs):.2e}  eager err "
      f"{float((eager - ref).abs().max() / ref.abs().max()):.2e}  replay==eager {torch.equal(out.float(), eager)}")
