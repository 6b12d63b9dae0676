"""Fixed cost of a timed CUDA-graph replay (events around graph.replay(), L2 flushed before) with
1, 2 and 4 trivial kernels, next to the C2 index build graphs."""
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
x = torch.zeros(256, device=dev)


def graphed(fn):
    side = torch.cuda.Stream()
    side.wait_stream(s)
    with torch.cuda.stream(side):
        fn()
    s.wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def timed(g, n=50):
    for _ in range(5):
        g.replay()
    ev = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(p.elapsed_time(q) for p, q in ev) * 1e3


for k in (1, 2, 4):
    print(f"{k} trivial kernel(s)         {timed(graphed(lambda k=k: [x.add_(1) for _ in range(k)])):6.1f} us")
w = dict(bench.WORKLOADS["bert_ffn1"], name="bert_ffn1")
A, B, live = bench.make_operands(w, seed=1234, device=dev)
print(f"build_index (1,768)        {timed(graphed(lambda: pit.build_index_from_tensor(A, (1, 768), 'm'))):6.1f} us")
