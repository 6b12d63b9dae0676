"""C4 dH = (dY . W2^T) * 1[H > 0] in H's live 1x32 micro-tiles: index build vs SDDMM time."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402
from paper_2301_10936_b200.sddmm import output_indexes_from_tensor, run_sddmm_like  # noqa: E402
from paper_2301_10936_b200.sddmm import _OutputSpec, run_sddmm  # noqa: E402

dev = torch.device("cuda", 0)
T, F, D = 4096, 8192, 2048
for zr in (0.9, 0.99):
    g = torch.Generator(device=dev).manual_seed(1)
    keep = torch.rand((T, F // 32), device=dev, generator=g) >= zr
    H = (torch.relu(torch.randn((T, F), device=dev, generator=g)) * keep.repeat_interleave(32, dim=1)).to(torch.bfloat16)
    dY = torch.randn((T, D), device=dev, dtype=torch.bfloat16, generator=g)
    W2 = torch.randn((F, D), device=dev, dtype=torch.bfloat16, generator=g) * 0.02
    flush = torch.empty(bench.FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    out = torch.zeros_like(H)
    ix = output_indexes_from_tensor(H, (1, 32))
    t_fine = bench._graph_ms(lambda: pit.build_index_from_tensor(H, (1, 32), "k"), flush, 10)
    t_unit = bench._graph_ms(lambda: pit.build_index_from_tensor(H, (128, 64), "k"), flush, 10)
    t_sd = bench._graph_ms(lambda: run_sddmm(dY, W2.t(), _OutputSpec(H.shape, (1, 32)), out=out, gate=H, indexes=ix), flush, 10)
    print(f"zero {zr}: fine index {t_fine:.3f} ms, unit index {t_unit:.3f} ms, sddmm {t_sd:.3f} ms, units {ix[0].total}")
