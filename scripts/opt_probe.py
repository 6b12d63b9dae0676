"""C4 weight-gradient product at 99% activation sparsity (pit:k, micro (32,1) on H^T) for ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2301_10936_b200 as pit  # noqa: E402

dev = torch.device("cuda", 0)
zr = float(sys.argv[1]) if len(sys.argv) > 1 else 0.99
tokens, d_ff, d_model = 4096, 8192, 2048
g = torch.Generator(device=dev).manual_seed(11)
keep = torch.rand((tokens, d_ff // 32), device=dev, generator=g) >= zr
H = torch.relu(torch.randn((tokens, d_ff), device=dev, dtype=torch.bfloat16, generator=g))
H.mul_(keep.repeat_interleave(32, dim=1).to(torch.bfloat16))
dY = torch.randn((tokens, d_model), device=dev, dtype=torch.bfloat16, generator=g)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
e = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=d_ff, k=tokens, n=d_model))
plan = pit.forced_plan(e, "k", reg, tile_shape=(32, 64, 32))
idx = pit.build_index_from_tensor(H, (1, 32), "m").transposed()
for _ in range(3):
    pit.run_matmul_with_index(plan, pit.DenseTensor(H.t()), pit.DenseTensor(dY), idx)
torch.cuda.synchronize()
print("total", idx.total, "max count", int(idx.counts.max()))
