"""C5 MoE layer alone on one GPU (16384 tokens x 128 experts, d 768 -> 3072 -> 768): per-kernel
launch list under ncu, or a CUDA-event time of the layer."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2301_10936_b200.moe import SwitchMoE  # noqa: E402

dev = torch.device("cuda", 0)
T, E, D, F = 16384, 128, 768, 3072
g = torch.Generator(device=dev).manual_seed(0)
w1 = torch.randn((E, D, F), device=dev, dtype=torch.bfloat16, generator=g) * 0.02
w2 = torch.randn((E, F, D), device=dev, dtype=torch.bfloat16, generator=g) * 0.02
x = torch.randn((T, D), device=dev, dtype=torch.bfloat16, generator=g)
logits = torch.randn((T, E), device=dev, dtype=torch.float32, generator=g)
moe = SwitchMoE(w1, w2, E)
for _ in range(3):
    moe.forward(x, logits)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    moe.forward(x, logits)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"MoE layer {ms:.4f} ms  {T / (ms * 1e-3) / 1e6:.1f} M tokens/s  weights {2 * E * D * F * 2 / (ms * 1e-3) / 1e12:.2f} TB/s")
