"""Small launches of the CTA-pair tcgen05 kernels for compute-sanitizer (racecheck / memcheck):
rowgemm2 (dense), spmm_gk2 (256x1 pit:k), rowgemm2t (grouped MoE FFN), K3s (high-sparsity pit:m).
    compute-sanitizer --tool racecheck python scripts/race_kernels.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2301_10936_b200 as pit  # noqa: E402
from paper_2301_10936_b200.moe import SwitchMoE  # noqa: E402

dev = torch.device("cuda", 0)
torch.manual_seed(0)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
for t in ((128, 64, 256), (256, 64, 256), (16, 32, 128)):
    if reg.get("matmul", t) is None:
        reg.register(pit.TileKernelDescriptor("matmul", t, "race"))


def plan(m, k, n, axis, tile):
    return pit.forced_plan(pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n)),
                           axis, reg, tile_shape=tile)


A = torch.randn((512, 256), device=dev, dtype=torch.bfloat16)
B = torch.randn((256, 512), device=dev, dtype=torch.bfloat16)
pit.run_sparse_matmul(plan(512, 256, 512, "dense", (128, 64, 256)), pit.DenseTensor(A), pit.DenseTensor(B), None)
At = (torch.randn((512, 512), device=dev, dtype=torch.bfloat16) * (torch.rand((512, 2), device=dev) > 0.5)
      .repeat_interleave(256, dim=1).to(torch.bfloat16)).t()
idx = pit.build_index_from_tensor(At, (256, 1), "k")
pit.run_matmul_with_index(plan(512, 512, 512, "k", (256, 64, 256)), pit.DenseTensor(At), pit.DenseTensor(B.repeat(2, 1)), idx)
keep = torch.rand((1024, 2048 // 32), device=dev) >= 0.995
H = (torch.relu(torch.randn((1024, 2048), device=dev)) * keep.repeat_interleave(32, dim=1)).to(torch.bfloat16)
W = torch.randn((2048, 384), device=dev, dtype=torch.bfloat16)
pit.run_matmul_with_index(plan(1024, 2048, 384, "m", (16, 32, 128)), pit.DenseTensor(H), pit.DenseTensor(W),
                          pit.build_index_from_tensor(H, (1, 32), "m"))
# column-axis detection (slab kernel, plain-store and atomic modes), the occupancy union, the 32x1
# gathered-K kernel (slot-index rotation) and the SDDMM with its two output indexes
from paper_2301_10936_b200.sddmm import run_sddmm_like  # noqa: E402

for micro in ((1, 32), (128, 64), (4, 8), (1, 256)):
    pit.build_index_from_tensor(H, micro, "k")
pit.build_index_from_tensor(H, (1, 32), "m").union_coords()
A32 = (torch.randn((512, 1024), device=dev, dtype=torch.bfloat16) * (torch.rand((512 // 32, 1024), device=dev) > 0.9)
       .repeat_interleave(32, dim=0).to(torch.bfloat16)).t().contiguous().t()
pit.run_matmul_with_index(plan(512, 1024, 1024, "k", (32, 64, 32)), pit.DenseTensor(A32),
                          pit.DenseTensor(torch.randn((1024, 1024), device=dev, dtype=torch.bfloat16)),
                          pit.build_index_from_tensor(A32, (32, 1), "k"))
run_sddmm_like(torch.randn((1024, 384), device=dev, dtype=torch.bfloat16), W.t(), H, (1, 32), gate=H)
w1 = torch.randn((8, 256, 512), device=dev, dtype=torch.bfloat16) * 0.05
w2 = torch.randn((8, 512, 256), device=dev, dtype=torch.bfloat16) * 0.05
moe = SwitchMoE(w1, w2, 8)
moe.forward(torch.randn((1024, 256), device=dev, dtype=torch.bfloat16), torch.randn((1024, 8), device=dev))
torch.cuda.synchronize()
print("race_kernels done")
