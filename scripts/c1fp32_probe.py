"""BASELINE configs[0] (1024^3 fp32, 32x1 @ 90%) step for a warm ncu kernel list / graph timing."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402

dev = torch.device("cuda", 0)
w = dict(bench.C1_1024, name="c1_fp32_1024")
g = torch.Generator(device=dev).manual_seed(3)
keep = torch.rand((w["K"], w["M"] // 32), device=dev, generator=g) >= w["zero"]
At = torch.randn((w["K"], w["M"]), device=dev, dtype=torch.float32, generator=g)
At.mul_(keep.repeat_interleave(32, dim=1).float())
A = At.t()
B = torch.randn((w["K"], w["N"]), device=dev, dtype=torch.float32, generator=g)
plan = bench.make_plan(w)
eff = 2.0 * w["N"] * int(keep.sum().item()) * 32
step = lambda: bench.pit_run(plan, A, B, w)  # noqa: E731
C = step()
ref = A.double() @ B.double()
print(f"rel err {float((C.double() - ref).norm() / ref.norm()):.2e}")
if "--ncu" in sys.argv:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    sys.exit(0)
flush = torch.empty(bench.FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
ms = bench._graph_ms(step, flush, 30)
print(f"step {ms * 1e3:.1f} us  {eff / ms / 1e9:.2f} TFLOP/s")
idx = pit.build_index_from_tensor(A, (32, 1), "k")
ms = bench._graph_ms(lambda: pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx), flush, 30)
print(f"spmm only {ms * 1e3:.1f} us")
