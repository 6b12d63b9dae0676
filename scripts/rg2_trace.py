"""Timeline of rowgemm2 (pair 0) from PIT_DIAG globaltimer stamps (needs a diagnostic build:
scripts/build_alt.sh WT diag with PIT_NVCC_DEFS=-DPIT_DIAG=1, then PIT_LIB_PATH=build_alt/libpit_diag.so).
    python scripts/rg2_trace.py [M K N]"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2301_10936_b200 as pit  # noqa: E402
from paper_2301_10936_b200 import _lib  # noqa: E402

bert = "--bert" in sys.argv
argv = [a for a in sys.argv[1:] if not a.startswith("--")]
m, k, n = (int(x) for x in (argv[:3] if len(argv) >= 3 else (2634, 768, 3072)))
dev = torch.device("cuda", 0)
lib = _lib.load()
reg = pit.register_builtin_kernels(include_b200_tiles=True)
A = torch.randn((m, k), device=dev, dtype=torch.bfloat16)
B = torch.randn((k, n), device=dev, dtype=torch.bfloat16)
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))
plan = pit.forced_plan(expr, "dense", reg, tile_shape=(128, 64, 256))
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
if bert:  # the C2 step's pit:m product over gathered live rows (PIT_SMALL_SINGLE=0 for the pair kernel)
    import bench

    w = dict(bench.WORKLOADS["bert_ffn1"], name="bert_ffn1")
    A, B, _ = bench.make_operands(w, seed=1234, device=dev)
    plan = bench.make_plan(w)
    idx = pit.build_index_from_tensor(A, w["micro"], w["axis"])
for _ in range(3):
    flush.zero_()
    if bert:
        pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx)
    else:
        pit.run_sparse_matmul(plan, pit.DenseTensor(A), pit.DenseTensor(B), None)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 1024)()
lib.pit_debug_gk2_trace(buf)
t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
entry = t[768:1024][t[768:1024] > 0]
t0 = entry.min()
print(f"CTA entry spread {(entry.max() - t0) / 1e3:.2f} us over {entry.size} CTAs; setup done +{(t[767] - t0) / 1e3:.2f} us")
rel = lambda v: (v - t0) / 1e3 if v > 0 else float("nan")  # noqa: E731
print("stage  prod_issue  relay0_full  relay1_full  mma_full   (us from first CTA entry)")
for j in range(0, 40):
    print(f"{j:5d} {rel(t[j]):10.2f} {rel(t[128 + j]):10.2f} {rel(t[384 + j]):10.2f} {rel(t[256 + j]):10.2f}")
print("unit  mma_start  epi_tmem_full  epi_done")
for u in range(8):
    if t[512 + u] or t[576 + u]:
        print(f"{u:4d} {rel(t[512 + u]):10.2f} {rel(t[576 + u]):10.2f} {rel(t[640 + u]):10.2f}")
