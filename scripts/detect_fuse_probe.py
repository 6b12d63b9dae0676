"""K1 detection (+ compaction) as a CUDA graph of the public call, L2 flushed before each replay,
mean of 50: C1's 128 MiB operand, the 512 MiB index-build case and C2's padded BERT rows. Run with
PIT_DETECT_FUSE / PIT_DETECT_BALANCE = 0 / 1 for same-box A/B."""
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402
from paper_2301_10936_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
s = torch.cuda.current_stream()
flush = torch.empty(bench.FLUSH_BYTES // 4, dtype=torch.float32, device=dev)


def graph_us(fn, n=50):
    side = torch.cuda.Stream()
    side.wait_stream(s)
    with torch.cuda.stream(side):
        for _ in range(2):
            fn()
    s.wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    k0 = _lib.kernel_launches()
    with torch.cuda.graph(g):
        fn()
    k = _lib.kernel_launches() - k0
    for _ in range(3):
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
    return statistics.mean(x.elapsed_time(y) for x, y in ev) * 1e3, k


tag = f"FUSE={os.environ.get('PIT_DETECT_FUSE', '1')} BALANCE={os.environ.get('PIT_DETECT_BALANCE', '1')}"
g = torch.Generator(device="cuda").manual_seed(7)
for side_ in (8192, 16384):
    keep = torch.rand((side_, side_ // 32), device=dev, generator=g) >= 0.9
    At = torch.randn((side_, side_), device=dev, dtype=torch.bfloat16, generator=g)
    At.mul_(keep.repeat_interleave(32, dim=1).to(torch.bfloat16))
    A = At.t()
    del keep
    t, k = graph_us(lambda: pit.build_index_from_tensor(A, (32, 1), "k"))
    nbytes = side_ * side_ * 2
    print(f"{tag}  {side_}^2 (32,1) k   {t:7.1f} us  {nbytes / t / 1e3:7.1f} GB/s  launches {k}")
    del A, At
w = dict(bench.WORKLOADS["bert_ffn1"], name="bert_ffn1")
A, B, live = bench.make_operands(w, seed=1234, device=dev)
t, k = graph_us(lambda: pit.build_index_from_tensor(A, (1, 768), "m"))
print(f"{tag}  BERT 4096x768 (1,768) m   {t:7.1f} us  launches {k}")
plan = bench.make_plan(w)
t, k = graph_us(lambda: bench.pit_run(plan, A, B, w))
print(f"{tag}  BERT step detect+pit:m   {t:7.1f} us  launches {k}")
