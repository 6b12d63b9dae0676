"""C3 attention step (pit:k (128,1) over column-major P, index from the device block mask) for a
warm per-kernel ncu list."""
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
if reg.get("matmul", (128, 64, 256)) is None:
    reg.register(pit.TileKernelDescriptor("matmul", (128, 64, 256), "a"))
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=seq, k=seq, n=hd))
plan = pit.forced_plan(expr, "k", reg, tile_shape=(128, 64, 256))
Pk = pit.stack_slices(P, plan)
del P
for _ in range(4):
    pit.run_batched_matmul_with_index(plan, Pk, V, pit.build_index(ann, (128, 1), "k"))
torch.cuda.synchronize()
