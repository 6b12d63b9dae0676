"""Seeded random sweep of the operator surface on the GPU against the CPU oracle.

Each case draws a shape (ragged and aligned), an operand dtype (fp32 FFMA path, bf16 / fp16
tensor-core paths), a PIT axis with a micro-tile, an annotation block granularity that need not
align with the micro-tile, a zero ratio from fully dead to fully live, and a route:
  * annotation route: ``run_sparse_matmul(plan, A, B, ann)`` (executor.py:519-537);
  * value route: ``build_index_from_tensor`` on the device operand + ``run_matmul_with_index``
    (index.py:164-173, executor.py:464-516), index dump compared with the oracle's.
Checks: the index (canonical dump, index.py:185-195), the product against the oracle's f64
evaluation of the same (rounded) inputs — 1e-5 normwise for fp32 (verify_close), 1e-2 for bf16 /
fp16 (max_rel_error) — and zero-completeness: M-blocks (pit:k) or rows (pit:m) with no live
micro-tile are exact zeros (test_executor.py:153-165).
"""

import os

import numpy as np
import pytest

from oracle import pit_oracle as orc

pytestmark = pytest.mark.gpu

MATMUL = "C[m,n] += A[m,k] * B[k,n]"
SCALE = int(os.environ.get("PIT_FUZZ_SCALE", "1"))  # PIT_FUZZ_SCALE=k: k times the cases (bug hunts)
N_CASES = 96 * SCALE


def _draw(cid):
    rng = np.random.default_rng(9000 + cid)
    dtype = rng.choice(["float32", "bfloat16", "bfloat16", "float16"])
    axis = rng.choice(["m", "k"])
    big = rng.random() < 0.35

    def ext():
        if big:
            return int(rng.choice([256, 384, 512, 640, 1024, 1000, 777, 1536]))
        return int(rng.integers(1, 300))

    m, k, n = ext(), ext(), ext()
    if dtype != "float32" and rng.random() < 0.7:
        n = max(8, n // 8 * 8)  # mostly 16-byte rows; the rest exercise ragged N
    if axis == "k":
        t = int(rng.choice([8, 16, 24, 32, 64, 128, 256]))
        tile = (t, 64, 256)
    else:
        t = int(rng.choice([16, 32, 64, 128]))
        tile = (128, t, 256)
    if dtype == "float32" and rng.random() < 0.5:
        tile = (32, 64, 32) if axis == "k" else (16, 32, 128)
    gran = (int(rng.choice([1, 2, 4, 8, 16, 32])), int(rng.choice([1, 2, 4, 8, 16, 32])))
    zero = float(rng.choice([0.0, 0.3, 0.8, 0.95, 0.99, 1.0]))
    route = rng.choice(["annotation", "values"])
    return dict(dtype=dtype, axis=axis, m=m, k=k, n=n, tile=tile, gran=gran, zero=zero, route=route,
                seed=int(rng.integers(1 << 30)))


@pytest.mark.parametrize("cid", range(N_CASES))
def test_random_case_matches_oracle(cid):
    import torch

    import paper_2301_10936_b200 as pit

    c = _draw(cid)
    m, k, n, axis, tile = c["m"], c["k"], c["n"], c["axis"], c["tile"]
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, f"fz{tile[0]}x{tile[1]}"))
    expr = pit.bind_extents(pit.parse_expr(MATMUL), dict(m=m, k=k, n=n))
    plan = pit.forced_plan(expr, axis, reg, tile_shape=tile)
    micro = tuple(plan.micro_tile)
    ann = pit.random_annotation((m, k), c["gran"], c["zero"], seed=c["seed"])
    rng = np.random.default_rng(c["seed"])
    A = rng.standard_normal((m, k)).astype(np.float32) * ann.materialize(np.float32)
    B = rng.standard_normal((k, n)).astype(np.float32)
    dt = getattr(torch, c["dtype"])
    Ad = torch.from_numpy(A).to(dt).cuda()
    if axis == "k":
        Ad = Ad.t().contiguous().t()
    Bd = torch.from_numpy(B).to(dt).cuda()
    Ar = Ad.double().cpu().numpy()
    Br = Bd.double().cpu().numpy()

    if c["route"] == "annotation":
        C = pit.run_sparse_matmul(plan, pit.DenseTensor(Ad), pit.DenseTensor(Bd), ann).array
        counts, groups = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, micro, axis)
    else:
        idx = pit.build_index_from_tensor(Ad, micro, axis)
        counts, groups = orc.build_index_from_values(Ar, micro, axis)
        assert pit.dump_index(idx) == orc.dump_index(micro, axis, counts, groups), c
        C = pit.run_matmul_with_index(plan, pit.DenseTensor(Ad), pit.DenseTensor(Bd), idx).array
    # A is zero outside its live micro-tiles, so the sparse product equals the dense f64 product
    ref = orc.dense_reference_f64(Ar, Br)
    assert C.is_cuda and C.dtype == dt and tuple(C.shape) == (m, n), c
    got = C.double().cpu().numpy()
    assert np.isfinite(got).all(), c
    if c["dtype"] == "float32":
        assert orc.verify_close(got, ref), (c, orc.max_rel_error(got, ref))
    else:
        assert orc.max_rel_error(got, ref) <= 1e-2, (c, orc.max_rel_error(got, ref))
    # zero-completeness
    if axis == "k":
        t0 = micro[0]
        for g in np.nonzero(np.asarray(counts) == 0)[0]:
            assert np.all(got[g * t0:(g + 1) * t0] == 0.0), (c, g)
    else:
        live = np.zeros(m, bool)
        for grp in groups:
            live[np.asarray(grp, dtype=np.int64)] = True
        assert np.all(got[~live] == 0.0), c


@pytest.mark.parametrize("cid", range(24 * SCALE))
def test_random_batched_case_matches_per_slice_oracle(cid):
    """Batched pit:k / pit:m (one launch over per-slice indexes, the prevalent-axis loop of
    README.md:152-155) with a random batch, shape, micro-tile and per-slice zero ratio."""
    import torch

    import paper_2301_10936_b200 as pit

    rng = np.random.default_rng(7100 + cid)
    batch = int(rng.integers(1, 5))
    axis = rng.choice(["m", "k"])
    m, k = int(rng.choice([128, 256, 384, 200, 96])), int(rng.choice([64, 128, 320, 512, 250]))
    n = int(rng.choice([64, 96, 128, 200, 256, 512]))
    dt = rng.choice([torch.bfloat16, torch.float16])
    t = int(rng.choice([8, 32, 128] if axis == "k" else [16, 32, 64]))
    tile = (t, 64, 256) if axis == "k" else (128, t, 256)
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, f"fzb{tile[0]}x{tile[1]}"))
    expr = pit.bind_extents(pit.parse_expr(MATMUL), dict(m=m, k=k, n=n))
    plan = pit.forced_plan(expr, axis, reg, tile_shape=tile)
    gran = (int(rng.choice([1, 4, 32])), int(rng.choice([1, 4, 32])))
    anns = [pit.random_annotation((m, k), gran, float(rng.choice([0.0, 0.5, 0.9, 0.99, 1.0])),
                                  seed=int(rng.integers(1 << 30))) for _ in range(batch)]
    A = np.stack([rng.standard_normal((m, k)).astype(np.float32) * a.materialize() for a in anns])
    B = rng.standard_normal((batch, k, n)).astype(np.float32)
    A3 = pit.stack_slices(torch.from_numpy(A).to(dt).cuda(), plan)
    B3 = torch.from_numpy(B).to(dt).cuda()
    stats = pit.ExecStats()
    try:
        C3 = pit.run_sparse_batched_matmul(plan, A3, B3, anns, stats=stats)
    except pit.ExecError as e:  # a stacked index needs slices on whole blocks and micro-tiles
        assert "multiple of the granularity" in str(e) and (m % gran[0] or m % plan.micro_tile[0]), (cid, e)
        return
    assert tuple(C3.shape) == (batch, m, n) and C3.dtype == dt
    Ar, Br, Cr = A3.double().cpu().numpy(), B3.double().cpu().numpy(), C3.double().cpu().numpy()
    launches = 0
    for b in range(batch):
        ref = orc.dense_reference_f64(Ar[b], Br[b])
        assert orc.max_rel_error(Cr[b], ref) <= 1e-2, (cid, b)
        if not anns[b].packed.any():
            assert np.all(Cr[b] == 0.0), (cid, b)
        launches += pit.plan_launches(plan, anns[b])
    assert stats.launches == launches


@pytest.mark.parametrize("cid", range(24 * SCALE))
def test_random_sddmm_case_matches_oracle(cid):
    """Output-sparse SDDMM (§8(f)3) over a random shape, output micro-tile and zero ratio: live
    micro-tiles hold A.B, dead ones keep ``out``'s sentinel."""
    import torch

    import paper_2301_10936_b200 as pit
    from paper_2301_10936_b200.sddmm import run_sddmm

    rng = np.random.default_rng(7300 + cid)
    M = int(rng.choice([1, 60, 128, 300, 512, 1000]))
    N = int(rng.choice([8, 64, 136, 512, 1024]))
    K = int(rng.choice([8, 16, 64, 72, 128, 256]))
    gran = (int(rng.choice([1, 2, 16, 32, 64, 128])), int(rng.choice([8, 16, 32, 64, 128])))
    zero = float(rng.choice([0.0, 0.5, 0.9, 0.99, 1.0]))
    dt = rng.choice([torch.bfloat16, torch.float16])
    A = torch.from_numpy(rng.standard_normal((M, K)).astype(np.float32)).to(dt).cuda()
    Bt = torch.from_numpy(rng.standard_normal((N, K)).astype(np.float32)).to(dt).cuda()
    ann = pit.random_annotation((M, N), gran, zero, seed=int(rng.integers(1 << 30)))
    out = torch.full((M, N), float("nan"), dtype=dt, device="cuda")
    run_sddmm(A, Bt.t(), ann, out=out)
    got = out.double().cpu().numpy()
    ref, live = orc.sddmm(A.double().cpu().numpy(), Bt.double().cpu().numpy().T,
                          (ann.tensor_shape, ann.granularity, ann.packed), np.full(got.shape, np.nan))
    assert np.isnan(got[~live]).all(), cid
    if live.any():
        assert orc.max_rel_error(got[live], ref[live]) <= 1e-2, cid


@pytest.mark.parametrize("cid", range(24 * SCALE))
def test_random_reduce_sum_case_matches_oracle(cid):
    """run_sparse_reduce_sum (executor.py:540-613) on a random shape / annotation / plan axis
    (pit:l, pit:p, dense) and dtype against the oracle; rows with no live element are exact zeros."""
    import paper_2301_10936_b200 as pit

    rng = np.random.default_rng(7500 + cid)
    p_, l_ = int(rng.integers(1, 400)), int(rng.integers(1, 700))
    axis = rng.choice(["l", "p", "dense"])
    dt = rng.choice([np.float32, np.float64])
    gran = (int(rng.choice([1, 2, 8])), int(rng.choice([1, 4, 16, 64])))
    ann = pit.random_annotation((p_, l_), gran, float(rng.choice([0.0, 0.5, 0.9, 1.0])),
                                seed=int(rng.integers(1 << 30)))
    A = (rng.standard_normal((p_, l_)) * ann.materialize(np.float64)).astype(dt)
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    expr = pit.bind_extents(pit.parse_expr("C[p] += A[p,l]"), dict(p=p_, l=l_))
    plan = pit.forced_plan(expr, str(axis), reg)
    C = pit.run_sparse_reduce_sum(plan, pit.DenseTensor.from_array(A), None if axis == "dense" else ann)
    got = np.asarray(C.array, dtype=np.float64)
    ref = orc.reduce_sum(A.astype(np.float64), (ann.tensor_shape, ann.granularity, ann.packed), str(axis),
                         plan.tile.tile_shape, np.float64)
    assert got.shape == (p_,) and orc.verify_close(got, ref), (cid, orc.max_rel_error(got, ref))
    if axis != "dense":
        assert np.all(got[~A.astype(bool).any(axis=1)] == 0.0), cid


@pytest.mark.parametrize("cid", range(24 * SCALE))
def test_random_sread_swrite_case_matches_oracle(cid):
    """SRead / SWrite (executor.py:170-264) on a random operand, micro-tile, axis, group, start
    offset and tile shape (partial and edge tiles included): tile, assigned and accumulated
    destinations bitwise equal to the oracle's."""
    import paper_2301_10936_b200 as pit

    rng = np.random.default_rng(7700 + cid)
    s0, s1 = int(rng.integers(1, 200)), int(rng.integers(1, 200))
    axis = rng.choice(["m", "k"])
    micro = (1, int(rng.choice([1, 4, 16, 32]))) if axis == "m" else (int(rng.choice([1, 4, 16, 32])), 1)
    d = 0 if axis == "m" else 1
    src = (rng.standard_normal((s0, s1)) * (rng.random((s0, s1)) < 0.3)).astype(np.float32)
    idx = pit.build_index(pit.from_mask(src, (1, 1)), micro, axis)
    counts, groups = orc.build_index(*orc.mask_to_ann(src != 0, (1, 1)), micro, axis)
    g = int(rng.integers(0, idx.n_groups))
    start = int(rng.integers(0, max(int(counts[g]), 1)))
    t_d = micro[d]
    n_slots = int(rng.integers(1, 9))
    other = micro[1 - d] if rng.random() < 0.7 else micro[1 - d] + int(rng.integers(1, 4))
    tshape = (n_slots * t_d, other) if d == 0 else (other, n_slots * t_d)
    tile = np.full(tshape, 9.0, np.float32)
    want_tile = tile.copy()
    n_ref = orc.sread(src, groups, micro, d, g, want_tile, start=start)
    assert pit.sread(src, idx, g, tile, start=start) == n_ref
    np.testing.assert_array_equal(tile, want_tile)
    for acc in (False, True):
        dst, want = np.ones_like(src), np.ones_like(src)
        assert pit.swrite(tile, dst, idx, g, start=start, accumulate=acc) == \
            orc.swrite(want_tile, want, groups, micro, d, g, start=start, accumulate=acc)
        np.testing.assert_array_equal(dst, want)


@pytest.mark.parametrize("cid", range(32 * SCALE))
def test_random_detection_special_values(cid):
    """K1 value-route detection (index.py:164-173) on random shapes, micro-tiles, dtypes and layouts
    with the special values of Appendix A.4 planted: -0.0 is zero; NaN, +-inf and subnormals are
    live. Canonical dump equal to the oracle's."""
    import torch

    import paper_2301_10936_b200 as pit

    rng = np.random.default_rng(7900 + cid)
    r, c = int(rng.integers(1, 700)), int(rng.integers(1, 700))
    dt = rng.choice([torch.float32, torch.float64, torch.bfloat16, torch.float16])
    axis = rng.choice(["m", "k"])
    t = int(rng.choice([1, 2, 3, 8, 16, 32, 64, 128, 256]))
    micro = (1, t) if axis == "m" else (t, 1)
    if rng.random() < 0.3:
        micro = (int(rng.choice([2, 4, 8])), t) if axis == "m" else (t, int(rng.choice([2, 4, 8])))
    x = np.zeros((r, c), np.float64)
    live = rng.random((r, c)) < float(rng.choice([0.0, 0.001, 0.02, 0.3]))
    x[live] = rng.standard_normal(int(live.sum()))
    tiny = {torch.float32: 1e-45, torch.float64: 5e-324, torch.bfloat16: 1e-40, torch.float16: 6e-8}[dt]
    for val in (-0.0, np.nan, np.inf, -np.inf, tiny, -tiny):
        n = int(rng.integers(0, 4))
        x[rng.integers(0, r, n), rng.integers(0, c, n)] = val
    xd = torch.from_numpy(x).to(dt).cuda()
    if rng.random() < 0.5:
        xd = xd.t().contiguous().t()  # column-major storage
    xr = xd.double().cpu().numpy()  # the values as stored (rounding / flush of the narrow types)
    idx = pit.build_index_from_tensor(xd, micro, axis)
    counts, groups = orc.build_index_from_values(xr, micro, axis)
    assert pit.dump_index(idx) == orc.dump_index(micro, axis, counts, groups), (cid, r, c, dt, micro, axis)


@pytest.mark.parametrize("cid", range(16 * SCALE))
def test_random_numpy_case_matches_oracle(cid):
    """The reference's own contract, numpy in / numpy out (f32 / f64), through run_sparse_matmul and
    build_index_from_tensor + run_matmul_with_index on host arrays; every fourth case has a B large
    enough (>= 32 MiB) for the pinned, slab-pipelined host path."""
    import paper_2301_10936_b200 as pit

    rng = np.random.default_rng(8100 + cid)
    dt = rng.choice([np.float32, np.float64])
    axis = rng.choice(["m", "k"])
    if cid % 4 == 3:
        m, k, n = int(rng.choice([64, 200])), 2048, 4096 if dt == np.float32 else 2048
    else:
        m, k, n = (int(rng.integers(1, 400)) for _ in range(3))
    tile = (32, 64, 32) if axis == "k" else (16, 32, 128)
    reg = pit.register_builtin_kernels()
    expr = pit.bind_extents(pit.parse_expr(MATMUL), dict(m=m, k=k, n=n))
    plan = pit.forced_plan(expr, str(axis), reg, tile_shape=tile)
    ann = pit.random_annotation((m, k), (int(rng.choice([1, 4, 32])), int(rng.choice([1, 4, 32]))),
                                float(rng.choice([0.0, 0.5, 0.9, 1.0])), seed=int(rng.integers(1 << 30)))
    A = (rng.standard_normal((m, k)) * ann.materialize(np.float64)).astype(dt)
    B = rng.standard_normal((k, n)).astype(dt)
    At = pit.DenseTensor.from_array(A, layout=plan.sparse_layout)
    if rng.random() < 0.5:
        C = pit.run_sparse_matmul(plan, At, pit.DenseTensor(B), ann).array
    else:
        idx = pit.build_index_from_tensor(At.array, plan.micro_tile, str(axis))
        C = pit.run_matmul_with_index(plan, At, pit.DenseTensor(B), idx).array
    assert isinstance(C, np.ndarray) and C.dtype == dt and C.shape == (m, n), cid
    ref = orc.dense_reference_f64(A.astype(np.float64), B.astype(np.float64))
    assert orc.verify_close(C.astype(np.float64), ref), (cid, orc.max_rel_error(C, ref))
