"""C2 BERT FFN1 breakdown: our captured step and its pieces vs cuBLAS (padded and live rows only).
   python scripts/bert_probe.py [--ncu]   (--ncu: a few eager steps for a launch list, no timing)"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402
from paper_2301_10936_b200.graph import CapturedSparseMatmul  # noqa: E402

dev = torch.device("cuda", 0)
w = dict(bench.WORKLOADS["bert_ffn1"], name="bert_ffn1")
A, B, live = bench.make_operands(w, seed=1234, device=dev)
plan = bench.make_plan(w)
eff = 2.0 * w["N"] * live
rows = live // w["K"]
if "--ncu" in sys.argv:
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=rows, k=w["K"], n=w["N"]))
    dplan = pit.forced_plan(expr, "dense", reg, tile_shape=(128, 64, 256))
    Al = torch.randn((rows, w["K"]), device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        bench.pit_run(plan, A, B, w)
        pit.run_sparse_matmul(dplan, pit.DenseTensor(Al), pit.DenseTensor(B), None)
        torch.matmul(Al, B)
    torch.cuda.synchronize()
    sys.exit(0)
flush = torch.empty(bench.FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()


def timed(fn, n=30):
    for _ in range(5):
        fn()
    ev = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.mean(x.elapsed_time(y) for x, y in ev) * 1e3  # mean: event timestamps are ~2 us quanta


def graphed(fn):
    side = torch.cuda.Stream()
    side.wait_stream(s)
    with torch.cuda.stream(side):
        for _ in range(2):
            fn()
    s.wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g.replay


cap = CapturedSparseMatmul(plan, A, B)
print(f"live rows {rows} of {w['M']}; effective {eff / 1e9:.2f} GFLOP")
t = timed(cap.replay)
print(f"pit step (graph)            {t:7.1f} us  {eff / t / 1e6:7.1f} TFLOP/s eff")
t = timed(graphed(lambda: pit.build_index_from_tensor(A, (1, 768), "m")))
print(f"index build only (graph)    {t:7.1f} us")
Al = torch.randn((rows, w["K"]), device=dev, dtype=torch.bfloat16)
for name, a in (("cuBLAS padded 4096", A), ("cuBLAS live rows", Al)):
    t = timed(graphed(lambda a=a: torch.matmul(a, B)))
    print(f"{name:28s}{t:7.1f} us  {eff / t / 1e6:7.1f} TFLOP/s eff")
reg = pit.register_builtin_kernels(include_b200_tiles=True)
for m_ in (rows, w["M"]):
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m_, k=w["K"], n=w["N"]))
    dplan = pit.forced_plan(expr, "dense", reg, tile_shape=(128, 64, 256))
    a = Al if m_ == rows else A
    t = timed(graphed(lambda a=a, dplan=dplan: pit.run_sparse_matmul(dplan, pit.DenseTensor(a), pit.DenseTensor(B), None)))
    print(f"pit dense plan M={m_:5d}       {t:7.1f} us  {2.0 * m_ * w['K'] * w['N'] / t / 1e6:7.1f} TFLOP/s")
