"""Where the e2e (host-buffer) step spends its time: H2D bandwidth, the pipelined B/C path alone."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402

w = dict(bench.WORKLOADS["pitk_c1_8192"], name="pitk_c1_8192")
dev = torch.device("cuda", 0)
A, B, live = bench.make_operands(w, 1234, dev)
plan = bench.make_plan(w)
Ah = torch.empty(A.t().shape, dtype=A.dtype, pin_memory=True)
Ah.copy_(A.t())
Bh = torch.empty(B.shape, dtype=B.dtype, pin_memory=True)
Bh.copy_(B)
Ch = torch.empty(B.shape, dtype=B.dtype, pin_memory=True)


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


h2d = t(lambda: Ah.to("cuda", non_blocking=True))
d2h = t(lambda: Ch.copy_(B, non_blocking=True))
Ad = Ah.to("cuda").t()
idx = pit.build_index_from_tensor(Ad, w["micro"], w["axis"])
pipe = t(lambda: pit.run_matmul_with_index(plan, pit.DenseTensor(Ad), pit.DenseTensor(Bh), idx))


def full():
    a = Ah.to("cuda", non_blocking=True).t()
    i = pit.build_index_from_tensor(a, w["micro"], w["axis"])
    pit.run_matmul_with_index(plan, pit.DenseTensor(a), pit.DenseTensor(Bh), i)


fu = t(full)
mb = Ah.numel() * 2 / 1e6
print(f"H2D 128 MiB: {h2d:.3f} ms = {mb / h2d:.1f} GB/s; D2H: {d2h:.3f} ms = {mb / d2h:.1f} GB/s")
print(f"pipelined B-up/SpMM/C-down (A resident): {pipe:.3f} ms; full e2e step: {fu:.3f} ms")

from paper_2301_10936_b200 import _lib  # noqa: E402

lib = _lib.load()
Bd = torch.empty_like(B)
K, N = Bh.shape
for slab in (1024, 2048, 8192):
    def up():
        s = torch.cuda.current_stream().cuda_stream
        for j0 in range(0, N, slab):
            lib.pit_copy2d_async(Bd.data_ptr() + j0 * 2, N * 2, Bh.data_ptr() + j0 * 2, N * 2, slab * 2, K, s)

    def down():
        s = torch.cuda.current_stream().cuda_stream
        for j0 in range(0, N, slab):
            lib.pit_copy2d_async(Ch.data_ptr() + j0 * 2, N * 2, Bd.data_ptr() + j0 * 2, N * 2, slab * 2, K, s)
    tu, td = t(up), t(down)
    print(f"2-D slabs of {slab} columns: H2D {mb / tu:.1f} GB/s, D2H {mb / td:.1f} GB/s")
