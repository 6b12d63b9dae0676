"""Split the C3 attention step per kernel (run under ncu --metrics gpu__time_duration.sum)."""
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
P = torch.randn((heads, seq, seq), device=dev, dtype=torch.bfloat16)
V = torch.randn((heads, seq, hd), device=dev, dtype=torch.bfloat16)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=seq, k=seq, n=hd))
plan_m = pit.forced_plan(expr, "m", reg, tile_shape=(128, 64, 256))
plan_k = pit.forced_plan(expr, "k", reg, tile_shape=(32, 64, 32))
Pk = pit.stack_slices(P, plan_k)
for _ in range(3):
    torch.cuda.nvtx.range_push("pit_m")
    im = pit.build_index(ann, (1, 64), "m")
    pit.run_batched_matmul_with_index(plan_m, P, V, im)
    torch.cuda.nvtx.range_pop()
    ik = pit.build_index(ann, (32, 1), "k")
    pit.run_batched_matmul_with_index(plan_k, Pk, V, ik)
torch.cuda.synchronize()
print("pit:m index total", im.total, "groups", im.n_groups, " pit:k total", ik.total)
plan_d = pit.forced_plan(expr, "dense", reg, tile_shape=(128, 64, 256))
for _ in range(2):
    pit.run_batched_matmul_with_index(plan_d, P, V, None)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    pit.run_batched_matmul_with_index(plan_d, P, V, None)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"dense batched P.V: {ms:.3f} ms, A stream {P.numel() * 2 / ms / 1e9:.0f} GB/s")
