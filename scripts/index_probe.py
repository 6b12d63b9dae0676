"""Run K1 (build_index_from_tensor) on a 16384^2 bf16 column-major tensor a few times (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2301_10936_b200 as pit  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = torch.Generator(device="cuda").manual_seed(99)
keep = torch.rand((side, side // 32), device="cuda", generator=g) >= 0.9
At = torch.randn((side, side), device="cuda", dtype=torch.bfloat16, generator=g)
At.mul_(keep.repeat_interleave(32, dim=1).to(torch.bfloat16))
A = At.t()
for _ in range(5):
    idx = pit.build_index_from_tensor(A, (32, 1), "k")
torch.cuda.synchronize()
print("total", idx.total)
