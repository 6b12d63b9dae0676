"""Stage / unit timeline of the single-CTA gathered-K kernel (CTA 0), PIT_GK2_DIAG bit 4 stamps.

    PIT_GK2_DIAG=16 python scripts/gk_trace.py [attn|c1]
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402
from paper_2301_10936_b200 import _lib  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "attn"
dev = torch.device("cuda", 0)
lib = _lib.load()
if which == "attn":
    heads, seq, hd = 12, 4096, 64
    blocks = bench.longformer_blocks(heads, seq, np.random.default_rng(3))
    ann = pit.from_bits(blocks.reshape(heads * seq // 32, seq // 64), (heads * seq, seq), (32, 64)).on_device(dev)
    P = torch.randn((heads, seq, seq), device=dev, dtype=torch.bfloat16)
    V = torch.randn((heads, seq, hd), device=dev, dtype=torch.bfloat16)
    reg = pit.register_builtin_kernels()
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=seq, k=seq, n=hd))
    plan = pit.forced_plan(expr, "k", reg, tile_shape=(32, 64, 32))
    Pk = pit.stack_slices(P, plan)
    ik = pit.build_index(ann, (32, 1), "k")
    run = lambda: pit.run_batched_matmul_with_index(plan, Pk, V, ik)  # noqa: E731
else:
    w = dict(bench.WORKLOADS["pitk_c1_8192"], name="pitk_c1_8192")
    A, B, live = bench.make_operands(w, 1234, dev)
    plan = bench.make_plan(w)
    idx = pit.build_index_from_tensor(A, w["micro"], w["axis"])
    run = lambda: pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx)  # noqa: E731
for _ in range(3):
    run()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 1024)()
lib.pit_debug_gk2_trace(buf)
t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(8, 128)
t0 = t[:6][t[:6] > 0].min()
rel = lambda e, j: (t[e, j] - t0) if t[e, j] else -1  # noqa: E731
print("stage   prod_issue   mma_full   mma_commit      | unit  mma_start  epi_start  epi_done")
for j in range(48):
    print(f"{j:5d} {rel(0, j):12d} {rel(1, j):10d} {rel(2, j):12d}      | {j:4d} {rel(3, j):10d} {rel(4, j):10d} {rel(5, j):9d}")
print("median ns between stage MMA starts:", np.median(np.diff(t[1, 1:100])))
