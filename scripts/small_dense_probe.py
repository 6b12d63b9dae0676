"""Small dense products (BERT-shaped) through the pit dense plan, for ncu (-k regex:rowgemm)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2301_10936_b200 as pit  # noqa: E402

dev = torch.device("cuda", 0)
m, k, n = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 768, 3072)))
reg = pit.register_builtin_kernels(include_b200_tiles=True)
tile = (128, 64, 256)
if reg.get("matmul", tile) is None:
    reg.register(pit.TileKernelDescriptor("matmul", tile, "probe"))
A = torch.randn((m, k), device=dev, dtype=torch.bfloat16)
B = torch.randn((k, n), device=dev, dtype=torch.bfloat16)
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))
plan = pit.forced_plan(expr, "dense", reg, tile_shape=tile)
for _ in range(5):
    pit.run_sparse_matmul(plan, pit.DenseTensor(A), pit.DenseTensor(B), None)
torch.cuda.synchronize()
