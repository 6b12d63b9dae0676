"""PIT sparse matmul on the GPU vs the CPU oracle.

Tolerances (north_star): fp32 path (FFMA, TF32 never used) within 1e-5 normwise of the
reference's f64 oracle (verify_close, executor.py:303-307); bf16 / fp16 tensor-core path within
1e-2 normwise (max_rel_error, executor.py:294-300) of the fp32-semantics oracle evaluated on the
same (bf16-rounded) inputs. Exact zeros are asserted bitwise.
"""

import numpy as np
import pytest

from oracle import pit_oracle as orc

pytestmark = pytest.mark.gpu

MATMUL = "C[m,n] += A[m,k] * B[k,n]"
BF16_TOL = 1e-2


def _pkg():
    import paper_2301_10936_b200 as pit

    return pit


def bound(m, k, n):
    pit = _pkg()
    return pit.bind_extents(pit.parse_expr(MATMUL), dict(m=m, k=k, n=n))


def _operands(m, k, n, ann, seed, dtype=np.float32):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, k)).astype(dtype) * ann.materialize(dtype)
    B = rng.standard_normal((k, n)).astype(dtype)
    return A, B


@pytest.mark.parametrize("axis,tile", [("m", (16, 32, 128)), ("k", (32, 64, 32)), ("dense", (32, 64, 32)),
                                        ("k", (8, 32, 128)), ("m", (32, 64, 32))])
@pytest.mark.parametrize("shape", [(64, 64, 64), (45, 70, 51), (128, 96, 160), (1, 200, 1), (200, 1, 1)])
def test_fp32_plans_match_oracle(axis, tile, shape):
    pit = _pkg()
    m, k, n = shape
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    ann = pit.random_annotation((m, k), (3, 2), 0.6, seed=m + k + n)
    A, B = _operands(m, k, n, ann, seed=7)
    plan = pit.forced_plan(bound(m, k, n), axis, reg, tile_shape=tile)
    At = pit.DenseTensor.from_array(A, layout=plan.sparse_layout)
    C = pit.run_sparse_matmul(plan, At, pit.DenseTensor.from_array(B), ann)
    oracle = orc.dense_reference_f64(A, B)
    assert orc.verify_close(C.array, oracle), orc.max_rel_error(C.array, oracle)
    if axis != "dense":
        ref = orc.run_sparse_matmul(A, B, (ann.tensor_shape, ann.granularity, ann.packed), axis, tile)
        assert orc.verify_close(C.array, ref)


def test_fp32_config1_1024_pit_k():
    """C1: 1024^3 fp32, random (32,1) micro-tile sparsity 90%, pit:k, tile 32x64x32."""
    pit = _pkg()
    m = k = n = 1024
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    ann = pit.random_annotation((m, k), (32, 1), 0.90, seed=1)
    A, B = _operands(m, k, n, ann, seed=1001)
    plan = pit.forced_plan(bound(m, k, n), "k", reg, tile_shape=(32, 64, 32))
    stats = pit.ExecStats()
    C = pit.run_sparse_matmul(plan, pit.DenseTensor.from_array(A, layout="col_major"), pit.DenseTensor.from_array(B),
                              ann, stats=stats)
    oracle = orc.dense_reference_f64(A, B)
    assert orc.verify_close(C.array, oracle)
    assert stats.launches == pit.plan_launches(plan, ann)
    assert stats.gathered_micro_tiles == pit.cover_count(ann, (32, 1))


def _bf16(x):
    import torch

    return torch.from_numpy(x).to(torch.bfloat16)


def _run_bf16(plan, A, B, ann, col_major):
    import torch

    pit = _pkg()
    At = _bf16(A).cuda()
    if col_major:
        At = At.t().contiguous().t()
    Bt = _bf16(B).cuda()
    C = pit.run_sparse_matmul(plan, pit.DenseTensor(At), pit.DenseTensor(Bt), ann)
    assert C.array.dtype == torch.bfloat16 and C.array.is_cuda
    Ar = At.float().cpu().numpy()
    Br = Bt.float().cpu().numpy()
    return C.array.float().cpu().numpy(), Ar, Br


@pytest.mark.parametrize("t0", [8, 16, 24, 32, 40, 64, 96, 128, 200, 256])
@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (512, 384, 520), (300, 200, 136)])
def test_bf16_pit_k_tensor_cores(t0, shape):
    pit = _pkg()
    m, k, n = shape
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    expr = bound(m, k, n)
    tile = (t0, 64, 256)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, f"t{t0}"))
    ann = pit.random_annotation((m, k), (t0, 1), 0.9, seed=t0 + m)
    A, B = _operands(m, k, n, ann, seed=t0)
    plan = pit.forced_plan(expr, "k", reg, tile_shape=tile)
    C, Ar, Br = _run_bf16(plan, A, B, ann, col_major=True)
    ref = orc.run_sparse_matmul(Ar, Br, (ann.tensor_shape, ann.granularity, ann.packed), "k", tile, np.float64)
    err = orc.max_rel_error(C, ref)
    assert err <= BF16_TOL, err
    # M-blocks whose group is empty are exact zeros
    counts, _ = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, (t0, 1), "k")
    for g in np.nonzero(counts == 0)[0]:
        assert np.all(C[g * t0 : (g + 1) * t0] == 0.0)


@pytest.mark.parametrize("t1", [16, 32, 64, 128])
@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (520, 384, 264), (300, 192, 100)])
def test_bf16_pit_m_tensor_cores(t1, shape):
    pit = _pkg()
    m, k, n = shape
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    tile = (128, t1, 256)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, f"m{t1}"))
    ann = pit.random_annotation((m, k), (1, t1), 0.9, seed=t1 + m)
    A, B = _operands(m, k, n, ann, seed=t1)
    plan = pit.forced_plan(bound(m, k, n), "m", reg, tile_shape=tile)
    C, Ar, Br = _run_bf16(plan, A, B, ann, col_major=False)
    ref = orc.run_sparse_matmul(Ar, Br, (ann.tensor_shape, ann.granularity, ann.packed), "m", tile, np.float64)
    err = orc.max_rel_error(C, ref)
    assert err <= BF16_TOL, err
    counts, groups = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, (1, t1), "m")
    live = set(np.concatenate(groups).tolist()) if groups else set()
    dead = [r for r in range(m) if r not in live]
    assert np.all(C[dead] == 0.0)


@pytest.mark.parametrize("t1", [16, 32])
@pytest.mark.parametrize("dead_rows", [0.0, 0.8])
@pytest.mark.parametrize("shape", [(1024, 2048, 512), (700, 416, 264)])
def test_bf16_pit_m_dead_micro_tiles_not_read(t1, dead_rows, shape):
    """pit:m reads only live (row, micro-column) tiles (SRead, executor.py:170-208): A carries
    non-zero data in every dead micro-tile. Scattered per-row patterns (union = ~all rows) run on
    contiguous row tiles with 64-deep K-blocks spanning 2-4 micro-columns; mostly-dead rows keep
    union-row tiles. Both must ignore the dead data."""
    pit = _pkg()
    m, k, n = shape
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    tile = (128, t1, 256)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, f"m{t1}"))
    rng = np.random.default_rng(t1 + m)
    mask = np.repeat(rng.random((m, -(-k // t1))) >= 0.9, t1, axis=1)[:, :k]
    mask[rng.random(m) < dead_rows] = False
    ann = pit.from_mask(mask, (1, t1))
    A = rng.standard_normal((m, k)).astype(np.float32)  # dense data: dead micro-tiles hold values too
    B = rng.standard_normal((k, n)).astype(np.float32)
    plan = pit.forced_plan(bound(m, k, n), "m", reg, tile_shape=tile)
    C, Ar, Br = _run_bf16(plan, A, B, ann, col_major=False)
    ref = orc.run_sparse_matmul(Ar, Br, (ann.tensor_shape, ann.granularity, ann.packed), "m", tile, np.float64)
    assert orc.max_rel_error(C, ref) <= BF16_TOL
    dead = ~mask.any(axis=1)
    assert np.all(C[dead] == 0.0)


@pytest.mark.parametrize("t1", [16, 32])
def test_bf16_pit_m_dead_neurons_skipped(t1):
    """Column-structured activation sparsity (dead neurons): only ~10% of the micro-columns hold any
    live row, but every row is live somewhere (union = all rows -> contiguous masked tiles on CTA
    pairs). Globally dead K-blocks are skipped; dead micro-tiles still hold data and must not count."""
    pit = _pkg()
    m, k, n = 1024, 4096, 512
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    tile = (128, t1, 256)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, f"m{t1}"))
    rng = np.random.default_rng(77 + t1)
    cols = rng.random(k // t1) < 0.1
    cols[0] = True
    mask = np.repeat((rng.random((m, k // t1)) < 0.5) & cols[None, :], t1, axis=1)
    mask[:, :t1] = True  # every row live in the first micro-column
    ann = pit.from_mask(mask, (1, t1))
    A = rng.standard_normal((m, k)).astype(np.float32)
    B = rng.standard_normal((k, n)).astype(np.float32)
    plan = pit.forced_plan(bound(m, k, n), "m", reg, tile_shape=tile)
    C, Ar, Br = _run_bf16(plan, A, B, ann, col_major=False)
    ref = orc.run_sparse_matmul(Ar, Br, (ann.tensor_shape, ann.granularity, ann.packed), "m", tile, np.float64)
    assert orc.max_rel_error(C, ref) <= BF16_TOL


def test_bf16_row_uniform_and_dense_bitwise():
    """Fully dense annotation through pit:m equals the dense plan bitwise (test_executor.py:178-186)."""
    pit = _pkg()
    m, k, n = 384, 512, 512
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    expr = bound(m, k, n)
    full = pit.from_mask(np.ones((m, k)), (1, 1))
    A, B = _operands(m, k, n, full, seed=3)
    sparse, _, _ = _run_bf16(pit.forced_plan(expr, "m", reg, tile_shape=(128, 64, 256)), A, B, full, False)
    dense, Ar, Br = _run_bf16(pit.forced_plan(expr, "dense", reg, tile_shape=(128, 64, 256)), A, B, None, False)
    assert np.array_equal(sparse, dense)
    assert orc.max_rel_error(dense, orc.dense_reference_f64(Ar, Br)) <= BF16_TOL


def test_bf16_row_uniform_bert_like():
    """C2-style: padded rows dead in every K-block (granularity (1,K))."""
    pit = _pkg()
    m, k, n = 4096, 768, 3072
    rng = np.random.default_rng(5)
    lengths = rng.integers(16, 129, size=32)
    rows = np.concatenate([np.arange(128) < L for L in lengths])
    mask = np.repeat(rows[:, None], k, axis=1)
    ann = pit.from_mask(mask, (1, k))
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    A, B = _operands(m, k, n, ann, seed=11)
    plan = pit.forced_plan(bound(m, k, n), "m", reg, tile_shape=(128, 64, 256))
    C, Ar, Br = _run_bf16(plan, A, B, ann, False)
    ref = orc.dense_reference_f64(Ar, Br)
    assert orc.max_rel_error(C, ref) <= BF16_TOL
    assert np.all(C[~rows] == 0.0)


def test_shuffled_slots_m_axis_bitwise_and_k_axis_close():
    pit = _pkg()
    m, k, n = 256, 256, 128
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    expr = bound(m, k, n)
    rng = np.random.default_rng(9)
    ann = pit.random_annotation((m, k), (1, 32), 0.5, seed=3)
    A, B = _operands(m, k, n, ann, seed=4)
    plan = pit.forced_plan(expr, "m", reg, tile_shape=(16, 32, 128))
    At, Bt = pit.DenseTensor.from_array(A), pit.DenseTensor.from_array(B)
    idx = pit.build_index(ann, plan.micro_tile, "m")
    ref = pit.run_matmul_with_index(plan, At, Bt, idx)
    sh = pit.canonicalize(idx)
    for g in range(sh.n_groups):
        c = sh.counts[g]
        sh.slots[g, :c] = rng.permutation(sh.slots[g, :c])
    got = pit.run_matmul_with_index(plan, At, Bt, sh)
    assert np.array_equal(got.array, ref.array)

    annk = pit.random_annotation((m, k), (32, 1), 0.5, seed=6)
    A64 = rng.standard_normal((m, k)) * annk.materialize(np.float64)
    B64 = rng.standard_normal((k, n))
    plank = pit.forced_plan(expr, "k", reg, tile_shape=(32, 64, 32))
    Ak = pit.DenseTensor.from_array(A64, layout="col_major", dtype=np.float64)
    Bk = pit.DenseTensor.from_array(B64, dtype=np.float64)
    idxk = pit.build_index(annk, plank.micro_tile, "k")
    refk = pit.run_matmul_with_index(plank, Ak, Bk, idxk)
    shk = pit.canonicalize(idxk)
    for g in range(shk.n_groups):
        c = shk.counts[g]
        shk.slots[g, :c] = rng.permutation(shk.slots[g, :c])
    gotk = pit.run_matmul_with_index(plank, Ak, Bk, shk)
    assert pit.max_rel_error(gotk, refk.array) <= 1e-12


def test_layout_and_operand_errors():
    pit = _pkg()
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    expr = bound(64, 64, 64)
    rng = np.random.default_rng(0)
    A = pit.DenseTensor.from_array(rng.standard_normal((64, 64)).astype(np.float32))
    B = pit.DenseTensor.from_array(rng.standard_normal((64, 64)).astype(np.float32))
    ann = pit.random_annotation((64, 64), (64, 1), 0.5, seed=2)
    with pytest.raises(pit.LayoutError, match="col_major"):
        pit.run_sparse_matmul(pit.forced_plan(expr, "k", reg), A, B, ann)
    with pytest.raises(pit.ExecError, match="needs a sparsity annotation"):
        pit.run_sparse_matmul(pit.forced_plan(expr, "m", reg), A, B, None)
    bad = pit.random_annotation((16, 64), (1, 1), 0.5, seed=0)
    with pytest.raises(pit.ExecError, match="annotation"):
        pit.run_sparse_matmul(pit.forced_plan(expr, "m", reg), A, B, bad)


def test_sread_swrite_round_trip_and_known_answers():
    pit = _pkg()
    bits = np.zeros((8, 4), bool)
    bits[[5, 1]] = True
    idx = pit.build_index(pit.from_mask(bits, (1, 1)), (1, 4), "m")
    src = np.zeros((8, 4), np.float32)
    src[5] = [1, 2, 3, 4]
    src[1] = [10, 20, 30, 40]
    buf = np.empty((2, 4), np.float32)
    assert pit.sread(src, idx, 0, buf) == 2
    assert {tuple(buf[0]), tuple(buf[1])} == {(1, 2, 3, 4), (10, 20, 30, 40)}
    pad = np.full((4, 4), 7.0, np.float32)
    idx1 = pit.build_index(pit.from_mask(np.eye(8, 4)[:, :] * 0 + (np.arange(8)[:, None] == 3), (1, 1)), (1, 4), "m")
    src2 = np.arange(32, dtype=np.float32).reshape(8, 4)
    assert pit.sread(src2, idx1, 0, pad) == 1
    assert np.array_equal(pad[0], src2[3]) and np.all(pad[1:] == 0.0)
    # column micro-tiles round trip
    rng = np.random.default_rng(1)
    s = np.zeros((6, 10), np.float32)
    s[:, 7] = rng.standard_normal(6)
    s[:, 2] = rng.standard_normal(6)
    idxc = pit.build_index(pit.from_mask(s, (1, 1)), (6, 1), "k")
    tb = np.empty((6, 4), np.float32)
    pit.sread(s, idxc, 0, tb)
    dst = np.zeros_like(s)
    pit.swrite(tb, dst, idxc, 0)
    assert np.array_equal(dst, s)
    # accumulate
    pit.swrite(tb, dst, idxc, 0, accumulate=True)
    assert np.allclose(dst, 2 * s)
    bad = pit.canonicalize(idx)
    bad.slots[0, 0] = 99
    with pytest.raises(pit.ExecError, match="out of range"):
        pit.sread(np.zeros((8, 4), np.float32), bad, 0, np.empty((2, 4), np.float32))
    with pytest.raises(pit.ExecError, match="group"):
        pit.sread(np.zeros((8, 4), np.float32), idx, 3, np.empty((2, 4), np.float32))


def test_dense_reference_f64_is_triple_loop():
    pit = _pkg()
    rng = np.random.default_rng(1234)
    A = rng.standard_normal((8, 8))
    B = rng.standard_normal((8, 8))
    assert np.array_equal(pit.run_dense_reference(A, B), orc.dense_reference_f64(A, B))


def test_captured_step_tracks_new_values():
    """CUDA-graph replay re-runs detection + SpMM on the buffers' current contents."""
    import torch

    pit = _pkg()
    from paper_2301_10936_b200.graph import CapturedSparseMatmul

    m, k, n = 512, 1024, 512
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    plan = pit.forced_plan(bound(m, k, n), "k", reg, tile_shape=(32, 64, 32))
    A = torch.zeros((k, m), dtype=torch.bfloat16, device="cuda").t()  # column-major buffer
    B = torch.randn((k, n), dtype=torch.bfloat16, device="cuda")
    step = CapturedSparseMatmul(plan, A, B)
    for seed in (1, 2):
        ann = pit.random_annotation((m, k), (32, 1), 0.9, seed=seed)
        Ah, _ = _operands(m, k, n, ann, seed=seed)
        A.copy_(torch.from_numpy(Ah).to(torch.bfloat16).cuda())
        C = step.replay().float().cpu().numpy()
        ref = orc.dense_reference_f64(A.float().cpu().numpy(), B.float().cpu().numpy())
        assert orc.max_rel_error(C, ref) <= BF16_TOL
    assert step.kernels_per_replay == 3


def test_sparse_reduce_sum_matches_reference_golden():
    """run_sparse_reduce_sum (executor.py:540-613) vs the reference's own outputs."""
    import json
    from pathlib import Path

    pit = _pkg()
    gold = Path(__file__).resolve().parent / "golden"
    data = np.load(gold / "reduce_cases.npz")
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    for c in json.loads((gold / "reduce_cases.json").read_text()):
        i = c["i"]
        p_, l_ = c["shape"]
        expr = pit.bind_extents(pit.parse_expr("C[p] += A[p,l]"), dict(p=p_, l=l_))
        ann = pit.from_ragged_lengths(c["lengths"], [p_, l_])
        plan = pit.forced_plan(expr, c["axis"], reg)
        stats = pit.ExecStats()
        C = pit.run_sparse_reduce_sum(plan, pit.DenseTensor.from_array(data[f"A{i}"]),
                                      ann if c["axis"] != "dense" else None, stats=stats)
        assert pit.verify_close(C, data[f"C{i}"].astype(np.float64)), i
        assert stats.launches == c["launches"] and stats.gathered_micro_tiles == c["gathered"], i
        if c["axis"] != "dense":
            empty = [r for r, n in enumerate(c["lengths"]) if n == 0]
            assert np.all(C.array[empty] == 0.0)
    A = np.random.default_rng(0).standard_normal((37, 91))
    np.testing.assert_allclose(pit.reduce_sum_reference(A), A.sum(axis=1), rtol=1e-12)
