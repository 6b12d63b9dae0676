"""rowgemm (gathered-M / dense / grouped) timings: dense 8192^3, dense 4096x3072x768, MoE layer.

    python scripts/rowgemm_probe.py [--ncu]   (with --ncu: one call each, for a launch list)
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2301_10936_b200 as pit  # noqa: E402
from paper_2301_10936_b200.moe import SwitchMoE  # noqa: E402

ncu = "--ncu" in sys.argv
dev = torch.device("cuda", 0)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
tile = (128, 64, 256)
if reg.get("matmul", tile) is None:
    reg.register(pit.TileKernelDescriptor("matmul", tile, "probe"))


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if ncu:
        fn()
        torch.cuda.synchronize()
        return float("nan")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for (m, k, n) in [(8192, 8192, 8192), (4096, 768, 3072), (4096, 3072, 768)]:
    A = torch.randn((m, k), device=dev, dtype=torch.bfloat16)
    B = torch.randn((k, n), device=dev, dtype=torch.bfloat16)
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))
    plan = pit.forced_plan(expr, "dense", reg, tile_shape=tile)
    ms = timed(lambda: pit.run_sparse_matmul(plan, pit.DenseTensor(A), pit.DenseTensor(B), None))
    ms_t = timed(lambda: torch.matmul(A, B))
    f = 2 * m * n * k
    print(f"dense {m}x{k}x{n}: pit {ms:.4f} ms = {f / ms / 1e9:.1f} TFLOP/s ; torch.matmul {ms_t:.4f} ms = {f / ms_t / 1e9:.1f}")

T, E, d, ff = 16384, 128, 768, 3072
g = torch.Generator(device=dev).manual_seed(7)
x = torch.randn((T, d), device=dev, dtype=torch.bfloat16, generator=g)
logits = torch.randn((T, E), device=dev, dtype=torch.float32, generator=g)
w1 = (torch.randn((E, d, ff), device=dev, generator=g) / d ** 0.5).to(torch.bfloat16)
w2 = (torch.randn((E, ff, d), device=dev, generator=g) / ff ** 0.5).to(torch.bfloat16)
layer = SwitchMoE(w1, w2, E)
ms = timed(lambda: layer(x, logits))
f = 2 * T * d * ff * 2
print(f"moe layer T={T}: {ms:.4f} ms = {T / ms / 1e3:.0f} k tokens/s, {f / ms / 1e9:.1f} TFLOP/s (expert FLOPs / layer time)")

# per-rank share of an 8-GPU expert-parallel layer: 16 local experts, 16384 received tokens
E8 = 16
w1b = (torch.randn((E8, d, ff), device=dev, generator=g) / d ** 0.5).to(torch.bfloat16)
w2b = (torch.randn((E8, ff, d), device=dev, generator=g) / ff ** 0.5).to(torch.bfloat16)
logits8 = torch.randn((T, E8), device=dev, dtype=torch.float32, generator=g)
layer8 = SwitchMoE(w1b, w2b, E8)
ms = timed(lambda: layer8(x, logits8))
print(f"moe layer T={T} E={E8} (EP8 per-rank proxy): {ms:.4f} ms = {T / ms / 1e3:.0f} k tokens/s, {f / ms / 1e9:.1f} TFLOP/s")
