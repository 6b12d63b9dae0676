"""C4-shaped pit:m with column-structured activation sparsity (dead neurons): H [4096, 8192] bf16,
only a fraction of the 32-wide neuron blocks ever fire, live blocks are 50% occupied per token.
Times build_index_from_tensor + run_matmul_with_index (device, CUDA events, L2 flushed)."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2301_10936_b200 as pit  # noqa: E402

T, F, D = 4096, 8192, 2048
dev = torch.device("cuda", 0)
for frac in (0.1, 0.3, 1.0):
    g = torch.Generator(device=dev).manual_seed(1)
    cols = torch.rand(F // 32, device=dev, generator=g) < frac
    cols[0] = True
    m = (torch.rand(T, F // 32, device=dev, generator=g) < 0.5) & cols[None, :]
    m[:, 0] = True
    H = torch.randn(T, F, device=dev, dtype=torch.bfloat16, generator=g) * m.repeat_interleave(32, 1).to(torch.bfloat16)
    W = torch.randn(F, D, device=dev, dtype=torch.bfloat16, generator=g)
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=T, k=F, n=D))
    if reg.get("matmul", (128, 32, 256)) is None:
        reg.register(pit.TileKernelDescriptor("matmul", (128, 32, 256), "m32"))
    plan = pit.forced_plan(expr, "m", reg, tile_shape=(128, 32, 256))
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    live = float((H != 0).sum())
    ts = []
    for i in range(8):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx = pit.build_index_from_tensor(H, (1, 32), "m")
        C = pit.run_matmul_with_index(plan, pit.DenseTensor(H), pit.DenseTensor(W), idx)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    ref = (H.float() @ W.float())
    err = float((C.array.float() - ref).abs().max() / ref.abs().max())
    print(f"live neuron blocks {frac:.0%}: step {ms:.4f} ms  {2 * D * live / (ms * 1e-3) / 1e12:.1f} TFLOP/s effective  err {err:.2e}")
