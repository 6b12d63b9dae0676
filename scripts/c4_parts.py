"""C4 step (OPT FFN2, 99% / 90% random 1x32 activation sparsity) broken into CUDA-graph parts
(L2 flushed before each replay, mean of 50): whole step, detection alone, forward alone, weight
gradient alone (index prebuilt)."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402

dev = torch.device("cuda", 0)
s = torch.cuda.current_stream()
flush = torch.empty(bench.FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
tokens, d_model, d_ff = 4096, 2048, 8192
reg = pit.register_builtin_kernels(include_b200_tiles=True)
fwd_e = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=tokens, k=d_ff, n=d_model))
bwd_e = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=d_ff, k=tokens, n=d_model))
plan_f = pit.forced_plan(fwd_e, "m", reg, tile_shape=(16, 32, 128))
plan_b = pit.forced_plan(bwd_e, "k", reg, tile_shape=(32, 64, 32))
g = torch.Generator(device=dev).manual_seed(11)
W2 = torch.randn((d_ff, d_model), device=dev, dtype=torch.bfloat16, generator=g) * 0.02
dY = torch.randn((tokens, d_model), device=dev, dtype=torch.bfloat16, generator=g)


def graphed(fn):
    side = torch.cuda.Stream()
    side.wait_stream(s)
    with torch.cuda.stream(side):
        for _ in range(2):
            fn()
    s.wait_stream(side)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    return gr


def timed(gr, n=50):
    for _ in range(5):
        gr.replay()
    ev = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        gr.replay()
        b.record(s)
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.mean(p.elapsed_time(q) for p, q in ev) * 1e3


for zr in [float(a) for a in sys.argv[1:]] or [0.99, 0.9]:
    keep = torch.rand((tokens, d_ff // 32), device=dev, generator=g) >= zr
    H = torch.relu(torch.randn((tokens, d_ff), device=dev, dtype=torch.bfloat16, generator=g))
    H.mul_(keep.repeat_interleave(32, dim=1).to(torch.bfloat16))
    idx = pit.build_index_from_tensor(H, (1, 32), "m")
    idt = idx.transposed()

    def step():
        ix = pit.build_index_from_tensor(H, (1, 32), "m")
        pit.run_matmul_with_index(plan_f, pit.DenseTensor(H), pit.DenseTensor(W2), ix)
        pit.run_matmul_with_index(plan_b, pit.DenseTensor(H.t()), pit.DenseTensor(dY), ix.transposed())

    print(f"zero {zr}")
    print(f"  whole step        {timed(graphed(step)):6.1f} us")
    print(f"  detection         {timed(graphed(lambda: pit.build_index_from_tensor(H, (1, 32), 'm'))):6.1f} us")
    print(f"  detect+transpose  {timed(graphed(lambda: pit.build_index_from_tensor(H, (1, 32), 'm').transposed())):6.1f} us")
    print(f"  forward           {timed(graphed(lambda: pit.run_matmul_with_index(plan_f, pit.DenseTensor(H), pit.DenseTensor(W2), idx))):6.1f} us")
    print(f"  weight gradient   {timed(graphed(lambda: pit.run_matmul_with_index(plan_b, pit.DenseTensor(H.t()), pit.DenseTensor(dY), idt))):6.1f} us")
