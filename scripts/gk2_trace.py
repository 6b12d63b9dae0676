"""Stage timeline of the CTA-pair gathered-K kernel (pair 0), from PIT_GK2_DIAG bit 4 stamps (needs a
diagnostic build: PIT_DIAG=1 python -m paper_2301_10936_b200._build --force).

    PIT_GK2_DIAG=16 python scripts/gk2_trace.py      (add 1/2/4 to drop MMA / copies / stores)
"""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402
from paper_2301_10936_b200 import _lib  # noqa: E402

w = dict(bench.WORKLOADS["pitk_256_8192"], name="pitk_256_8192")
dev = torch.device("cuda", 0)
lib = _lib.load()
A, B, live = bench.make_operands(w, 1234, dev)
plan = bench.make_plan(w)
idx = pit.build_index_from_tensor(A, w["micro"], w["axis"])
for _ in range(3):
    pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 1024)()
lib.pit_debug_gk2_trace(buf)
t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(8, 128)
t0 = t[:6][t[:6] > 0].min()
names = ["prod0 issue", "prod1 issue", "relay0 full", "relay1 full", "mma pair_full", "mma committed"]
print("stage " + " ".join(f"{n:>14s}" for n in names) + "   (ns from first stamp)")
for j in range(0, 40):
    print(f"{j:5d} " + " ".join(f"{(t[e, j] - t0) if t[e, j] else -1:14d}" for e in range(6)))
d = np.diff(t[4, 1:100])
print("median ns between MMA stage starts:", np.median(d), " diag", os.environ.get("PIT_GK2_DIAG"))
