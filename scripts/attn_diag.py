"""Time the C3 attention SpMM alone (pit:k (32,1) and pit:m (1,64) batched), index prebuilt."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402

dev = torch.device("cuda", 0)
heads, seq, hd = 12, 4096, 64
blocks = bench.longformer_blocks(heads, seq, np.random.default_rng(3))
ann = pit.from_bits(blocks.reshape(heads * seq // 32, seq // 64), (heads * seq, seq), (32, 64)).on_device(dev)
live = int(blocks.sum()) * 32 * 64
P = torch.randn((heads, seq, seq), device=dev, dtype=torch.bfloat16)
V = torch.randn((heads, seq, hd), device=dev, dtype=torch.bfloat16)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=seq, k=seq, n=hd))
plan_m = pit.forced_plan(expr, "m", reg, tile_shape=(128, 64, 256))
plan_k = pit.forced_plan(expr, "k", reg, tile_shape=(32, 64, 32))
Pk = pit.stack_slices(P, plan_k)
im = pit.build_index(ann, (1, 64), "m")
ik = pit.build_index(ann, (32, 1), "k")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


mk = t(lambda: pit.run_batched_matmul_with_index(plan_k, Pk, V, ik))
mm = t(lambda: pit.run_batched_matmul_with_index(plan_m, P, V, im))
bi = t(lambda: pit.build_index(ann, (32, 1), "k"))
f = 2.0 * hd * live
print(f"pit:k spmm {mk * 1e3:.1f} us ({f / mk / 1e9:.1f} TF)  pit:m spmm {mm * 1e3:.1f} us  build_index(k) {bi * 1e3:.1f} us"
      f"  groups with work {int((ik.counts > 0).sum()) if hasattr(ik, 'counts') else '?'}  total {ik.total}")

# wider query groups: union of adjacent query blocks' keys (Longformer windows overlap), bigger MMAs
for t0 in (64, 128):
    tile = (t0, 64, 256)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, f"attn{t0}"))
    pl = pit.forced_plan(expr, "k", reg, tile_shape=tile)
    Pt = pit.stack_slices(P, pl)
    ix = pit.build_index(ann, (t0, 1), "k")
    ms = t(lambda: pit.run_batched_matmul_with_index(pl, Pt, V, ix))
    bt = t(lambda: pit.build_index(ann, (t0, 1), "k"))
    print(f"pit:k ({t0},1): spmm {ms * 1e3:.1f} us ({f / ms / 1e9:.1f} TF effective), build_index {bt * 1e3:.1f} us, "
          f"covered/live = {ix.total * t0 / (live / 64):.3f}")
