"""High-sparsity pit:m path (csrc/pit_gm_sparse.cu: supergroup products with fp32 partial rows and an
ordered row reduction) on the GPU against an f64 reference: random (1,32) / (1,16) activation
sparsity at and around the device-side switch (live fraction 1/48), dead rows exactly zero, bitwise
repeatability (the reduction order is fixed), and the masked dense path beside it (PIT_GM_SPARSE=0
in a child process) agreeing within the bf16 tolerance.

Reference: _matmul_pit_m (executor.py:352-383) — per K-block group, the live rows' tile product is
scatter-accumulated into C.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import pit_oracle as orc

pytestmark = pytest.mark.gpu
BF16_TOL = 1e-2
ROOT = Path(__file__).resolve().parent.parent


def _case(tokens, d_ff, d_model, zero, t1=32, seed=0, dtype="bfloat16"):
    import torch

    import paper_2301_10936_b200 as pit

    dt = getattr(torch, dtype)
    g = torch.Generator(device="cuda").manual_seed(seed)
    keep = torch.rand((tokens, d_ff // t1), device="cuda", generator=g) >= zero
    H = torch.relu(torch.randn((tokens, d_ff), device="cuda", generator=g)).to(dt)
    H.mul_(keep.repeat_interleave(t1, dim=1).to(dt))
    W = (torch.randn((d_ff, d_model), device="cuda", generator=g) * 0.05).to(dt)
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    if reg.get("matmul", (16, t1, 128)) is None:
        reg.register(pit.TileKernelDescriptor("matmul", (16, t1, 128), "t"))
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=tokens, k=d_ff, n=d_model))
    plan = pit.forced_plan(expr, "m", reg, tile_shape=(16, t1, 128))
    idx = pit.build_index_from_tensor(H, (1, t1), "m")
    return pit, plan, idx, H, W, keep


@pytest.mark.parametrize("tokens,d_ff,d_model,zero,t1,dtype", [
    (4096, 8192, 2048, 0.99, 32, "bfloat16"),    # C4 at 99%: the sparse path
    (4096, 8192, 2048, 0.985, 32, "bfloat16"),   # still under the switch
    (1000, 2048, 384, 0.995, 32, "bfloat16"),    # ragged token count, narrow output
    (2048, 4096, 512, 0.995, 16, "bfloat16"),    # 16-wide micro-columns
    (2048, 4096, 1024, 0.99, 32, "float16"),     # fp16 operands
    (4096, 8192, 2048, 0.9, 32, "bfloat16"),     # 90%: the masked dense path (flag clear)
])
def test_pitm_high_sparsity_matches_f64(tokens, d_ff, d_model, zero, t1, dtype):
    import torch

    pit, plan, idx, H, W, keep = _case(tokens, d_ff, d_model, zero, t1, seed=tokens + d_model, dtype=dtype)
    poison = torch.full((tokens, d_model), float("nan"), dtype=H.dtype, device="cuda")
    del poison  # every row of C must be written (the allocator hands this block out next)
    C = pit.run_matmul_with_index(plan, pit.DenseTensor(H), pit.DenseTensor(W), idx).array
    ref = (H.double() @ W.double())
    got = C.double()
    assert not torch.isnan(got).any()
    dead = ~keep.any(dim=1)
    assert torch.all(got[dead] == 0)
    err = float((got - ref).norm() / ref.norm().clamp_min(1e-30))
    assert err <= BF16_TOL, err


def test_pitm_high_sparsity_repeatable_and_graph_safe():
    """The same call twice (and as a CUDA-graph replay after the values change) gives bitwise the
    eager result: the partial rows are summed in ascending supergroup order, no atomics."""
    import torch

    from paper_2301_10936_b200.graph import CapturedSparseMatmul

    pit, plan, idx, H, W, keep = _case(4096, 8192, 2048, 0.99, seed=3)
    C1 = pit.run_matmul_with_index(plan, pit.DenseTensor(H), pit.DenseTensor(W), idx).array.clone()
    C2 = pit.run_matmul_with_index(plan, pit.DenseTensor(H), pit.DenseTensor(W), idx).array
    assert torch.equal(C1, C2)
    cap = CapturedSparseMatmul(plan, H, W)
    g = torch.Generator(device="cuda").manual_seed(9)
    keep2 = torch.rand(keep.shape, device="cuda", generator=g) >= 0.99
    H.copy_(torch.relu(torch.randn(H.shape, device="cuda", generator=g)).to(H.dtype) *
            keep2.repeat_interleave(32, dim=1).to(H.dtype))
    out = cap.replay()
    idx2 = pit.build_index_from_tensor(H, (1, 32), "m")
    eager = pit.run_matmul_with_index(plan, pit.DenseTensor(H), pit.DenseTensor(W), idx2).array
    assert torch.equal(out, eager)


def test_pitm_sparse_path_agrees_with_masked_dense_path():
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2301_10936_b200 as pit
g = torch.Generator(device="cuda").manual_seed(5)
keep = torch.rand((2048, 4096 // 32), device="cuda", generator=g) >= 0.99
H = torch.relu(torch.randn((2048, 4096), device="cuda", generator=g)).to(torch.bfloat16)
H.mul_(keep.repeat_interleave(32, dim=1).to(torch.bfloat16))
W = (torch.randn((4096, 1024), device="cuda", generator=g) * 0.05).to(torch.bfloat16)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=2048, k=4096, n=1024))
plan = pit.forced_plan(expr, "m", reg, tile_shape=(16, 32, 128))
idx = pit.build_index_from_tensor(H, (1, 32), "m")
C = pit.run_matmul_with_index(plan, pit.DenseTensor(H), pit.DenseTensor(W), idx).array
np.save(sys.argv[1], C.float().cpu().numpy())
""" % str(ROOT)
    import tempfile

    outs = []
    for flag in ("1", "0"):
        f = tempfile.mktemp(suffix=".npy")
        r = subprocess.run([sys.executable, "-c", code, f], env=dict(os.environ, PIT_GM_SPARSE=flag),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert orc.max_rel_error(outs[0], outs[1].astype(np.float64)) <= BF16_TOL
    assert np.array_equal(outs[0] == 0, outs[1] == 0)
