"""C3 attention P.V, pit:k (128,1) variant alone: per-kernel device times (CUDA events) of the
index build from the block mask and the batched SpMM; runnable under ncu (-k regex:spmm_gk)."""
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
micro = int(sys.argv[1]) if len(sys.argv) > 1 else 128
blocks = bench.longformer_blocks(heads, seq, np.random.default_rng(3))
if len(sys.argv) > 2 and sys.argv[2] == "noglobalrow":  # probe: drop the global query block row
    blocks[:, 0, :] = blocks[:, 1, :]
ann = pit.from_bits(blocks.reshape(heads * seq // 32, seq // 64), (heads * seq, seq), (32, 64)).on_device(dev)
g = torch.Generator(device=dev).manual_seed(5)
emask = torch.from_numpy(blocks).to(dev).repeat_interleave(32, 1).repeat_interleave(64, 2)
P = torch.randn((heads, seq, seq), device=dev, dtype=torch.bfloat16, generator=g) * emask.to(torch.bfloat16)
del emask
V = torch.randn((heads, seq, hd), device=dev, dtype=torch.bfloat16, generator=g)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=seq, k=seq, n=hd))
tile = (micro, 64, 256)
if reg.get("matmul", tile) is None:
    reg.register(pit.TileKernelDescriptor("matmul", tile, "attn"))
plan = pit.forced_plan(expr, "k", reg, tile_shape=tile)
A3k = pit.stack_slices(P, plan)
ref = P[0].double() @ V[0].double()
del P
flush = torch.empty(bench.FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
idx = pit.build_index(ann, (micro, 1), "k")
O = pit.run_batched_matmul_with_index(plan, A3k, V, idx)
O = O.array if hasattr(O, "array") else O
err = float((O[0].double() - ref).abs().max() / ref.abs().max())
live = int(blocks.sum()) * 32 * 64
t_idx, t_mm = [], []
s = torch.cuda.current_stream()
for _ in range(10):
    flush.zero_()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(s)
    idx = pit.build_index(ann, (micro, 1), "k")
    e[1].record(s)
    pit.run_batched_matmul_with_index(plan, A3k, V, idx)
    e[2].record(s)
    torch.cuda.synchronize()
    t_idx.append(e[0].elapsed_time(e[1]))
    t_mm.append(e[1].elapsed_time(e[2]))
mm = statistics.median(t_mm)
gathered = int(idx.total) * (micro * 2 + hd * 2)
print(f"micro ({micro},1): index {statistics.median(t_idx):.4f} ms  spmm {mm:.4f} ms  "
      f"eff {2 * hd * live / (mm * 1e-3) / 1e12:.1f} TFLOP/s  total live k {int(idx.total)}  "
      f"gathered {gathered / 1e6:.1f} MB -> {gathered / (mm * 1e-3) / 1e9:.0f} GB/s  "
      f"ideal bytes {(live * 2 + 2 * heads * seq * hd * 2) / 1e6:.1f} MB  err {err:.2e}")
