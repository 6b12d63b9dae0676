"""numpy operands through run_sparse_matmul: staged-and-pipelined (now) vs synchronous staging (before)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2301_10936_b200 as pit  # noqa: E402
from paper_2301_10936_b200 import executor  # noqa: E402

m, k, n = 2048, 4096, 8192
reg = pit.register_builtin_kernels()
plan = pit.forced_plan(pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n)), "k", reg,
                       tile_shape=(32, 64, 32))
ann = pit.random_annotation((m, k), (32, 1), 0.9, seed=3)
rng = np.random.default_rng(1)
A = pit.DenseTensor.from_array((rng.standard_normal((m, k)) * ann.materialize(np.float32)).astype(np.float32), layout="col_major")
B = pit.DenseTensor.from_array(rng.standard_normal((k, n)).astype(np.float32))
for label, stage in (("pipelined", executor._stageable), ("synchronous", lambda b: False)):
    executor._stageable = stage
    pit.run_sparse_matmul(plan, A, B, ann)
    t = time.perf_counter()
    for _ in range(5):
        C = pit.run_sparse_matmul(plan, A, B, ann)
    print(f"{label:12s} {(time.perf_counter() - t) / 5 * 1e3:.1f} ms per call (B {B.array.nbytes >> 20} MiB numpy fp32)")
