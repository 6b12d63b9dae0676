"""C4 forward (OPT FFN2 H.W2 at random 1x32 activation sparsity) per-kernel probe.
    python scripts/c4_probe.py [zero_ratio] [--ncu]"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2301_10936_b200 as pit  # noqa: E402

zr = float(next((a for a in sys.argv[1:] if not a.startswith("--")), 0.99))
dev = torch.device("cuda", 0)
tokens, d_ff, d_model = 4096, 8192, 2048
g = torch.Generator(device=dev).manual_seed(11)
keep = torch.rand((tokens, d_ff // 32), device=dev, generator=g) >= zr
H = torch.relu(torch.randn((tokens, d_ff), device=dev, generator=g)).to(torch.bfloat16)
H.mul_(keep.repeat_interleave(32, dim=1).to(torch.bfloat16))
W2 = (torch.randn((d_ff, d_model), device=dev, generator=g) * 0.02).to(torch.bfloat16)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=tokens, k=d_ff, n=d_model))
plan = pit.forced_plan(expr, "m", reg, tile_shape=(16, 32, 128))
idx = pit.build_index_from_tensor(H, (1, 32), "m")
eff = 2.0 * d_model * int(keep.sum().item()) * 32
fn = lambda: pit.run_matmul_with_index(plan, pit.DenseTensor(H), pit.DenseTensor(W2), idx)  # noqa: E731
for _ in range(3):
    C = fn()
torch.cuda.synchronize()
ref = H.double() @ W2.double()
print(f"zero {zr}: live {keep.float().mean().item():.4f}, rel err {float((C.array.double() - ref).norm() / ref.norm()):.2e}")
if "--ncu" in sys.argv:
    sys.exit(0)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
ev = []
for _ in range(20):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    fn()
    b.record(s)
    ev.append((a, b))
torch.cuda.synchronize()
ms = statistics.mean(x.elapsed_time(y) for x, y in ev)
print(f"fwd eager {ms * 1e3:.1f} us  {eff / ms / 1e9:.1f} TFLOP/s effective")
