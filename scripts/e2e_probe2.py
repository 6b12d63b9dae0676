"""Where the e2e step's time goes: the public API on pinned host buffers vs its PCIe floor."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402

dev = torch.device("cuda", 0)
w = dict(bench.WORKLOADS["pitk_c1_8192"], name="pitk_c1_8192")
A, B, live = bench.make_operands(w, 1234, dev)
plan = bench.make_plan(w)
Ah = torch.empty(A.t().shape, dtype=A.dtype, pin_memory=True)
Ah.copy_(A.t())
Bh = torch.empty(B.shape, dtype=B.dtype, pin_memory=True)
Bh.copy_(B)


def once():
    Ad = Ah.to("cuda", non_blocking=True).t()
    idx = pit.build_index_from_tensor(Ad, w["micro"], w["axis"])
    return pit.run_matmul_with_index(plan, pit.DenseTensor(Ad), pit.DenseTensor(Bh), idx)


for _ in range(3):
    once()
torch.cuda.synchronize()
for n in (1, 5):
    t = time.perf_counter()
    for _ in range(n):
        once()
    torch.cuda.synchronize()
    print(f"once x{n}: {(time.perf_counter() - t) / n * 1e3:.3f} ms per call (wall)")
s = torch.cuda.current_stream()
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
e[0].record(s)
Ad = Ah.to("cuda", non_blocking=True).t()
e[1].record(s)
idx = pit.build_index_from_tensor(Ad, w["micro"], w["axis"])
e[2].record(s)
C = pit.run_matmul_with_index(plan, pit.DenseTensor(Ad), pit.DenseTensor(Bh), idx)
e[3].record(s)
torch.cuda.synchronize()
print(f"A upload {e[0].elapsed_time(e[1]):.3f} ms, detect {e[1].elapsed_time(e[2]):.3f} ms, pipelined B/SpMM/C {e[2].elapsed_time(e[3]):.3f} ms")
