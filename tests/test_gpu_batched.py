"""Batched PIT matmul over a prevalent axis (heads / slices): one launch
over slices stacked along M must equal the per-slice reference algorithm (independent index per
slice) — checked slice by slice against the oracle. Also the narrow-N (<= 128) tensor-core units."""

import numpy as np
import pytest

from oracle import pit_oracle as orc

pytestmark = pytest.mark.gpu
BF16_TOL = 1e-2


def _pit():
    import paper_2301_10936_b200 as pit

    return pit


def _bound(m, k, n):
    pit = _pit()
    return pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))


def _tile_for(reg, t0):
    pit = _pit()
    tile = (t0, 64, 256)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, f"t{t0}"))
    return tile


@pytest.mark.parametrize("t0", [8, 32, 128, 256])
@pytest.mark.parametrize("n", [64, 100, 300])
def test_batched_pit_k_bf16_matches_per_slice_oracle(t0, n):
    import torch

    pit = _pit()
    batch, m, k = 3, 256, 384
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    plan = pit.forced_plan(_bound(m, k, n), "k", reg, tile_shape=_tile_for(reg, t0))
    anns = [pit.random_annotation((m, k), (t0, 1), 0.85, seed=10 * t0 + b) for b in range(batch)]
    rng = np.random.default_rng(t0 + n)
    A = np.stack([rng.standard_normal((m, k)).astype(np.float32) * a.materialize() for a in anns])
    B = rng.standard_normal((batch, k, n)).astype(np.float32)
    A3 = pit.stack_slices(torch.from_numpy(A).to(torch.bfloat16).cuda(), plan)
    B3 = torch.from_numpy(B).to(torch.bfloat16).cuda()
    stats = pit.ExecStats()
    C3 = pit.run_sparse_batched_matmul(plan, A3, B3, anns, stats=stats)
    assert C3.shape == (batch, m, n) and C3.dtype == torch.bfloat16
    Ar, Br, Cr = A3.float().cpu().numpy(), B3.float().cpu().numpy(), C3.float().cpu().numpy()
    launches = 0
    for b in range(batch):
        ann = anns[b]
        ref = orc.run_sparse_matmul(Ar[b], Br[b], (ann.tensor_shape, ann.granularity, ann.packed), "k",
                                    plan.tile.tile_shape, np.float64)
        assert orc.max_rel_error(Cr[b], ref) <= BF16_TOL, b
        launches += pit.plan_launches(plan, ann)
    assert stats.launches == launches
    # one detection pass over the stacked operand gives the same stacked index
    idx = pit.build_batched_index_from_tensor(A3, plan.micro_tile, "k")
    ref_idx = pit.build_batched_index(anns, plan.micro_tile, "k")
    # standard-normal values inside live blocks are never exactly 0: the dumps must be equal
    assert pit.dump_index(idx) == pit.dump_index(ref_idx)


def test_batched_fp32_and_dense_slices():
    import torch

    pit = _pit()
    batch, m, k, n = 2, 64, 96, 40
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    rng = np.random.default_rng(5)
    anns = [pit.random_annotation((m, k), (32, 1), 0.7, seed=b) for b in range(batch)]
    A = np.stack([rng.standard_normal((m, k)).astype(np.float32) * a.materialize() for a in anns])
    B = rng.standard_normal((batch, k, n)).astype(np.float32)
    plan = pit.forced_plan(_bound(m, k, n), "k", reg, tile_shape=(32, 64, 32))
    C = pit.run_sparse_batched_matmul(plan, A, B, anns)  # host arrays: explicit stacking inside
    dense = pit.forced_plan(_bound(m, k, n), "dense", reg)
    Cd = pit.run_batched_matmul_with_index(dense, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), None)
    for b in range(batch):
        oracle = orc.dense_reference_f64(A[b], B[b])
        assert orc.verify_close(C[b], oracle)
        assert orc.verify_close(Cd[b].cpu().numpy(), oracle)


def test_batched_layout_is_never_converted_silently():
    import torch

    pit = _pit()
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    plan = pit.forced_plan(_bound(64, 64, 64), "k", reg, tile_shape=(32, 64, 32))
    A3 = torch.zeros((2, 64, 64), device="cuda")  # row-major slices, not stacked col-major
    with pytest.raises(pit.LayoutError, match="stack_slices"):
        pit.run_batched_matmul_with_index(plan, A3, torch.zeros((2, 64, 64), device="cuda"), None)


@pytest.mark.parametrize("t0", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("n", [64, 128, 72])
def test_narrow_n_units(t0, n):
    """N <= 128 runs 128-column units (attention P.V with head dim 64)."""
    import torch

    pit = _pit()
    m, k = 512, 1024
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    plan = pit.forced_plan(_bound(m, k, n), "k", reg, tile_shape=_tile_for(reg, t0))
    ann = pit.random_annotation((m, k), (t0, 1), 0.9, seed=t0 + n)
    rng = np.random.default_rng(n)
    A = rng.standard_normal((m, k)).astype(np.float32) * ann.materialize()
    B = rng.standard_normal((k, n)).astype(np.float32)
    At = torch.from_numpy(A).to(torch.bfloat16).cuda().t().contiguous().t()
    Bt = torch.from_numpy(B).to(torch.bfloat16).cuda()
    C = pit.run_sparse_matmul(plan, pit.DenseTensor(At), pit.DenseTensor(Bt), ann).array.float().cpu().numpy()
    ref = orc.run_sparse_matmul(At.float().cpu().numpy(), Bt.float().cpu().numpy(),
                                (ann.tensor_shape, ann.granularity, ann.packed), "k", plan.tile.tile_shape, np.float64)
    assert orc.max_rel_error(C, ref) <= BF16_TOL


@pytest.mark.parametrize("t1", [16, 32, 64])
@pytest.mark.parametrize("n", [40, 64, 300])
def test_batched_pit_m_bf16_matches_per_slice_oracle(t1, n):
    """Batched pit:m (rows x t1 micro-tiles, e.g. row-major attention P with 64-key blocks): one
    launch over uniform row groups; slice 1 is all-zero so its rows must come out exactly 0."""
    import torch

    pit = _pit()
    batch, m, k = 3, 320, 256
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    tile = (16, t1, 128)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, f"m{t1}"))
    plan = pit.forced_plan(_bound(m, k, n), "m", reg, tile_shape=tile)
    assert plan.micro_tile == (1, t1)
    ratios = [0.8, 1.0, 0.95]
    anns = [pit.random_annotation((m, k), (32, t1), r, seed=7 * t1 + b) for b, r in enumerate(ratios)]
    rng = np.random.default_rng(t1 * n)
    A = np.stack([rng.standard_normal((m, k)).astype(np.float32) * a.materialize() for a in anns])
    B = rng.standard_normal((batch, k, n)).astype(np.float32)
    A3 = pit.stack_slices(torch.from_numpy(A).to(torch.bfloat16).cuda(), plan)
    B3 = torch.from_numpy(B).to(torch.bfloat16).cuda()
    stats = pit.ExecStats()
    C3 = pit.run_sparse_batched_matmul(plan, A3, B3, anns, stats=stats)
    Ar, Br, Cr = A3.float().cpu().numpy(), B3.float().cpu().numpy(), C3.float().cpu().numpy()
    launches = 0
    for b in range(batch):
        ann = anns[b]
        ref = orc.run_sparse_matmul(Ar[b], Br[b], (ann.tensor_shape, ann.granularity, ann.packed), "m",
                                    tile, np.float64)
        if not np.any(ref):
            assert not np.any(Cr[b]), b
        else:
            assert orc.max_rel_error(Cr[b], ref) <= BF16_TOL, b
        launches += pit.plan_launches(plan, ann)
    assert stats.launches == launches
    assert not np.any(Cr[1]) and np.all(np.signbit(Cr[1]) == False)  # noqa: E712  exact +0.0


def test_pit_m_narrow_n_two_d():
    import torch

    pit = _pit()
    m, k, n = 1000, 512, 48
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    plan = pit.forced_plan(_bound(m, k, n), "m", reg, tile_shape=(16, 32, 128))
    ann = pit.random_annotation((m, k), (1, 32), 0.9, seed=2)
    rng = np.random.default_rng(2)
    A = rng.standard_normal((m, k)).astype(np.float32) * ann.materialize()
    B = rng.standard_normal((k, n)).astype(np.float32)
    At = torch.from_numpy(A).to(torch.bfloat16).cuda()
    Bt = torch.from_numpy(B).to(torch.bfloat16).cuda()
    C = pit.run_sparse_matmul(plan, pit.DenseTensor(At), pit.DenseTensor(Bt), ann).array.float().cpu().numpy()
    ref = orc.run_sparse_matmul(At.float().cpu().numpy(), Bt.float().cpu().numpy(),
                                (ann.tensor_shape, ann.granularity, ann.packed), "m", (16, 32, 128), np.float64)
    assert orc.max_rel_error(C, ref) <= BF16_TOL


@pytest.mark.parametrize("m,n", [(200, 300), (512, 264), (96, 520)])
def test_batched_dense_bf16_cta_pairs(m, n):
    """Dense batched slices run on CTA pairs (rowgemm2, 256-row pair tiles): slice heights that are
    not a multiple of 256 leave partial and empty pair halves; every slice must equal its product."""
    import torch

    pit = _pit()
    batch, k = 3, 192
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    tile = (128, 64, 256)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, "d128"))
    plan = pit.forced_plan(_bound(m, k, n), "dense", reg, tile_shape=tile)
    rng = np.random.default_rng(m + n)
    A = torch.from_numpy(rng.standard_normal((batch, m, k)).astype(np.float32)).to(torch.bfloat16).cuda()
    B = torch.from_numpy(rng.standard_normal((batch, k, n)).astype(np.float32)).to(torch.bfloat16).cuda()
    C = pit.run_sparse_batched_matmul(plan, pit.stack_slices(A, plan), B, None)
    ref = torch.bmm(A.double(), B.double())
    for b in range(batch):
        assert orc.max_rel_error(C[b].float().cpu().numpy(), ref[b].cpu().numpy()) <= BF16_TOL, b


@pytest.mark.parametrize("batch,m,n", [(4, 1024, 64), (1, 1000, 40), (2, 512, 64)])
def test_split_long_groups_narrow_n(batch, m, n):
    """Few, unequal groups (attention with global query rows): 128-row gathered-K groups longer than
    twice the mean are split over several CTAs and their fp32 partial tiles summed (split units).
    Result must match the per-slice oracle; empty groups stay exact zeros."""
    import torch

    pit = _pit()
    k, t0 = 4096, 128
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    plan = pit.forced_plan(_bound(m, k, n), "k", reg, tile_shape=_tile_for(reg, t0))
    rng = np.random.default_rng(m + n)
    mask = np.repeat(rng.random((batch, -(-m // t0), k)) >= 0.9, t0, axis=1)[:, :m]
    mask[:, :t0, :] = True                  # a global group per slice: every key live
    mask[:, t0 : 2 * t0, :] = False          # and an empty one
    A = rng.standard_normal((batch, m, k)).astype(np.float32) * mask
    B = rng.standard_normal((batch, k, n)).astype(np.float32)
    At = torch.from_numpy(A).to(torch.bfloat16).cuda()
    B3 = torch.from_numpy(B).to(torch.bfloat16).cuda()
    if batch > 1:
        A3 = pit.stack_slices(At, plan)
        idx = pit.build_batched_index_from_tensor(A3, (t0, 1), "k")
        C3 = pit.run_batched_matmul_with_index(plan, A3, B3, idx).float().cpu().numpy()
    else:
        A2 = At[0].t().contiguous().t()
        idx = pit.build_index_from_tensor(A2, (t0, 1), "k")
        C3 = pit.run_matmul_with_index(plan, pit.DenseTensor(A2), pit.DenseTensor(B3[0]), idx).array
        C3 = C3.float().cpu().numpy()[None]
    Ar, Br = At.float().cpu().numpy(), B3.float().cpu().numpy()
    for b in range(batch):
        ref = orc.dense_reference_f64(Ar[b], Br[b])
        assert orc.max_rel_error(C3[b], ref) <= BF16_TOL, b
        assert np.all(C3[b, t0 : 2 * t0] == 0.0)
    lib = pit._lib.load()
    assert lib.pit_spmm_workspace_bytes is not None
