"""Row-uniform pit:m (whole-row micro-tiles (1, K): BERT's padding removal, BASELINE configs[1]) on
the GPU: the fused detection + compaction launch, the packed-row CTA-pair GEMM and its in-kernel
clearing of dead rows, against the oracle / an f64 reference.

Indices bit-exact (equal counts and ordered slots); bf16 results within 1e-2 normwise (north_star);
rows no group names are exact zeros.
"""

import numpy as np
import pytest

from oracle import pit_oracle as orc

pytestmark = pytest.mark.gpu
BF16_TOL = 1e-2


def _pkg():
    import paper_2301_10936_b200 as pit

    return pit


def _plan(m, k, n, axis="m", tile=(128, 64, 256)):
    pit = _pkg()
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    if reg.get("matmul", tuple(tile)) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tuple(tile), "t"))
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))
    return pit.forced_plan(expr, axis, reg, tile_shape=tile)


@pytest.mark.parametrize("rows,cols,p_live", [(1, 64, 1.0), (31, 64, 0.5), (4096, 768, 0.6), (100003, 64, 0.3),
                                               (1 << 20, 8, 0.5), (5000, 256, 0.0), (5000, 256, 1.0)])
def test_fused_whole_row_detection_bit_exact(rows, cols, p_live):
    """One cooperative launch (detect + compact) for (1, >= C) micro-tiles: counts and the ordered
    row list equal the oracle's, from 1 row to 2^20 rows, all-dead and all-live included."""
    import torch

    pit = _pkg()
    rng = np.random.default_rng(rows + cols)
    live = rng.random(rows) < p_live
    v = torch.zeros((rows, cols), dtype=torch.bfloat16)
    hot = torch.from_numpy(np.nonzero(live)[0])
    col = torch.from_numpy(rng.integers(0, cols, size=hot.numel()))
    v[hot, col] = 1.5
    idx = pit.build_index_from_tensor(v.cuda(), (1, cols), "m")
    assert int(idx.counts[0]) == int(live.sum())
    np.testing.assert_array_equal(np.asarray(idx.group(0)), np.nonzero(live)[0])
    if rows <= 5000:
        counts, groups = orc.build_index_from_values(v.float().numpy(), (1, cols), "m")
        assert pit.dump_index(idx) == orc.dump_index((1, cols), "m", counts, groups)


@pytest.mark.parametrize("lengths_seed", [1, 2])
def test_bert_step_from_values_matches_f64(lengths_seed):
    """The C2 step exactly as bench.py runs it: detection from the activations, then the product
    (live rows packed, TMA-fed CTA-pair GEMM, dead rows cleared inside the GEMM)."""
    import torch

    pit = _pkg()
    m, k, n = 4096, 768, 3072
    rng = np.random.default_rng(lengths_seed)
    lengths = rng.integers(16, 129, size=m // 128)
    rows = np.concatenate([np.arange(128) < L for L in lengths])
    g = torch.Generator().manual_seed(lengths_seed)
    A = (torch.randn((m, k), generator=g) * torch.from_numpy(rows)[:, None]).to(torch.bfloat16).cuda()
    B = torch.randn((k, n), generator=g).to(torch.bfloat16).cuda()
    idx = pit.build_index_from_tensor(A, (1, k), "m")
    poison = torch.full((m, n), float("nan"), dtype=torch.bfloat16, device="cuda")
    del poison  # the caching allocator hands this block to the output next: every row must be written
    out = pit.run_matmul_with_index(_plan(m, k, n, tile=(128, k, 256)), pit.DenseTensor(A), pit.DenseTensor(B), idx)
    got = out.array.float().cpu().numpy()
    ref = (A.double() @ B.double()).cpu().numpy()
    assert orc.max_rel_error(got[rows], ref[rows]) <= BF16_TOL
    assert np.all(got[~rows] == 0.0) and not np.isnan(got).any()


@pytest.mark.parametrize("n_live,dtype", [(0, "bfloat16"), (1, "bfloat16"), (37, "bfloat16"), (255, "bfloat16"),
                                          (256, "bfloat16"), (257, "bfloat16"), (2000, "bfloat16"), (1500, "float16")])
def test_row_uniform_live_counts_and_poisoned_output(n_live, dtype):
    """Live-row counts around the 256-row pair tile and the 32-row store boxes; the output buffer is
    poisoned before the call and every row must come back finite (live) or exactly zero (dead)."""
    import torch

    pit = _pkg()
    m, k, n = 2048, 256, 384
    rng = np.random.default_rng(n_live)
    live = np.zeros(m, dtype=bool)
    live[rng.choice(m, size=n_live, replace=False)] = True
    dt = getattr(torch, dtype)
    A = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float32) * live[:, None]).to(dt).cuda()
    B = torch.from_numpy(rng.standard_normal((k, n)).astype(np.float32)).to(dt).cuda()
    idx = pit.build_index_from_tensor(A, (1, k), "m")
    poison = torch.full((m, n), float("nan"), dtype=dt, device="cuda")
    del poison  # the caching allocator hands this block to the output next
    C = pit.run_matmul_with_index(_plan(m, k, n, tile=(128, k, 256)), pit.DenseTensor(A), pit.DenseTensor(B), idx)
    got = C.array.float().cpu().numpy()
    ref = (A.double() @ B.double()).cpu().numpy()
    assert np.all(got[~live] == 0.0) and not np.isnan(got).any()
    if n_live:
        assert orc.max_rel_error(got[live], ref[live]) <= BF16_TOL


def test_row_uniform_matches_gather_path_bitwise():
    """Packing the live rows first changes where A comes from, not the arithmetic: bitwise equal to
    the cp.async row-gather kernel (PIT_GM_PACK=0 in a child process)."""
    import subprocess
    import sys
    from pathlib import Path

    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2301_10936_b200 as pit
m, k, n = 3000, 768, 1024
rng = np.random.default_rng(4)
live = rng.random(m) < 0.55
A = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float32) * live[:, None]).to(torch.bfloat16).cuda()
B = torch.from_numpy(rng.standard_normal((k, n)).astype(np.float32)).to(torch.bfloat16).cuda()
reg = pit.register_builtin_kernels(include_b200_tiles=True)
expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))
reg.register(pit.TileKernelDescriptor("matmul", (128, k, 256), "t"))
plan = pit.forced_plan(expr, "m", reg, tile_shape=(128, k, 256))
idx = pit.build_index_from_tensor(A, (1, k), "m")
C = pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx).array
np.save(sys.argv[1], C.view(torch.int16).cpu().numpy())
""" % str(Path(__file__).resolve().parent.parent)
    import os
    import tempfile

    outs = []
    for pack in ("1", "0"):
        f = tempfile.mktemp(suffix=".npy")
        env = dict(os.environ, PIT_GM_PACK=pack, PIT_SMALL_SINGLE="0")
        r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])
