"""K1 detection / index construction on the GPU vs the CPU oracle: bit-exact.

"Bit-exact" = equal counts and equal groups. The GPU compaction is
ordered, so groups are compared without canonicalization against the reference's workers=1
order (ascending).
"""

import numpy as np
import pytest

from oracle import pit_oracle as orc

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2301_10936_b200 as pit

    return pit


def assert_same_index(idx, counts, groups):
    np.testing.assert_array_equal(idx.counts, counts)
    for g in range(idx.n_groups):
        np.testing.assert_array_equal(idx.group(g), groups[g], err_msg=f"group {g}")


CASES = [
    # shape, granularity, micro, axis, zero ratio
    ((64, 64), (1, 1), (1, 8), "m", 0.7),
    ((64, 64), (1, 1), (8, 1), "k", 0.7),
    ((45, 70), (3, 2), (1, 32), "m", 0.6),
    ((45, 70), (3, 2), (16, 1), "k", 0.6),
    ((1024, 1024), (32, 1), (32, 1), "k", 0.9),
    ((1024, 1024), (1, 32), (1, 32), "m", 0.9),
    ((1000, 777), (2, 3), (5, 7), "m", 0.95),
    ((1000, 777), (2, 3), (5, 7), "k", 0.3),
    ((1, 1), (1, 1), (1, 1), "m", 0.4),
    ((200, 1), (1, 1), (16, 1), "k", 0.4),
    ((1, 200), (1, 1), (1, 32), "m", 0.4),
    ((4096, 4096), (2, 1), (16, 1), "k", 0.95),
    ((4096, 4096), (1, 64), (1, 64), "m", 0.99),
]


@pytest.mark.parametrize("shape,gran,micro,axis,ratio", CASES)
def test_build_index_annotation_matches_oracle(shape, gran, micro, axis, ratio):
    pit = _pkg()
    ann = pit.random_annotation(shape, gran, ratio, seed=shape[0] * 7 + shape[1])
    idx = pit.build_index(ann, micro, axis)
    counts, groups = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, micro, axis)
    assert_same_index(idx, counts, groups)


def test_build_index_sweep_matches_oracle():
    pit = _pkg()
    rng = np.random.default_rng(4)
    for trial in range(120):
        shape = (int(rng.integers(1, 300)), int(rng.integers(1, 300)))
        gran = (int(rng.integers(1, 6)), int(rng.integers(1, 6)))
        micro = (int(rng.integers(1, 40)), int(rng.integers(1, 40)))
        axis = "m" if rng.integers(2) else "k"
        ann = pit.random_annotation(shape, gran, float(rng.choice([0.0, 0.3, 0.7, 0.95, 1.0])), seed=trial)
        idx = pit.build_index(ann, micro, axis)
        counts, groups = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, micro, axis)
        assert_same_index(idx, counts, groups)


FUSED_BITS_CASES = [
    # power-of-two geometry with coordinate blocks >= 32 coordinates wide: bitmap words derived from
    # the packed bits inside the compaction launch (bits_compact_pow2_kernel)
    ((4096, 4096), (32, 64), (128, 1), "k", 0.8),   # C3's key index of a 32x64 block mask
    ((4096, 4096), (32, 64), (32, 1), "k", 0.8),
    ((1000, 3000), (32, 64), (64, 2), "k", 0.7),    # ragged extents, t1 = 2
    ((2048, 1024), (64, 32), (1, 1), "m", 0.5),
    ((777, 333), (128, 4), (4, 8), "m", 0.3),
    ((256, 131072), (32, 64), (128, 1), "k", 0.9),  # two long groups: split over blockIdx.y
    ((96, 65536), (32, 128), (32, 4), "k", 0.0),    # fully live
    ((96, 65536), (32, 128), (32, 4), "k", 1.0),    # fully dead
]


@pytest.mark.parametrize("shape,gran,micro,axis,ratio", FUSED_BITS_CASES)
def test_build_index_fused_bits_route_matches_oracle(shape, gran, micro, axis, ratio):
    pit = _pkg()
    ann = pit.random_annotation(shape, gran, ratio, seed=shape[0] * 3 + shape[1])
    idx = pit.build_index(ann, micro, axis)
    counts, groups = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, micro, axis)
    assert_same_index(idx, counts, groups)
    # the bitmap the fused launch stores is the one the two-launch route writes
    occ = idx.occupancy_words().cpu().numpy().view(np.uint32)
    ref_occ = np.zeros(occ.shape, np.uint32)
    for g, grp in enumerate(groups):
        grp = np.asarray(grp, dtype=np.int64)
        np.bitwise_or.at(ref_occ[g], grp // 32, (np.uint32(1) << (grp % 32).astype(np.uint32)))
    np.testing.assert_array_equal(occ, ref_occ)


def test_build_index_fused_bits_sweep_matches_oracle():
    pit = _pkg()
    rng = np.random.default_rng(11)
    for trial in range(60):
        axis = "m" if rng.integers(2) else "k"
        cg = int(rng.choice([32, 64, 128]))           # coordinate-axis granularity
        ct = int(rng.choice([1, 2, 4]))
        ct = min(ct, cg // 32)                         # coordinate blocks >= 32 coordinates
        gg, gt = int(rng.choice([1, 2, 8, 32])), int(rng.choice([1, 4, 16, 128]))
        cs, gs = int(rng.integers(1, 5000)), int(rng.integers(1, 600))
        shape, gran, micro = ((cs, gs), (cg, gg), (ct, gt)) if axis == "m" else ((gs, cs), (gg, cg), (gt, ct))
        ann = pit.random_annotation(shape, gran, float(rng.choice([0.0, 0.5, 0.9, 1.0])), seed=100 + trial)
        idx = pit.build_index(ann, micro, axis)
        counts, groups = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, micro, axis)
        assert_same_index(idx, counts, groups)


DTYPES = ["float32", "float64", "bfloat16", "float16", "uint8", "bool"]


def _values(shape, density, rng):
    v = rng.standard_normal(shape).astype(np.float32)
    v[rng.random(shape) >= density] = 0.0
    return v


def _torch_values(v, dtype, col_major):
    import torch

    t = torch.from_numpy(v)
    if dtype == "bool":
        t = t != 0
    elif dtype == "uint8":
        t = (t != 0).to(torch.uint8) * 3
    else:
        t = t.to(getattr(torch, dtype))
    t = t.cuda()
    if col_major:
        t = t.t().contiguous().t()
    return t


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("col_major", [False, True])
@pytest.mark.parametrize(
    "shape,micro,axis",
    [((256, 512), (1, 32), "m"), ((256, 512), (32, 1), "k"), ((300, 200), (3, 5), "m"), ((300, 200), (7, 2), "k"),
     ((512, 1024), (1, 64), "m"), ((1024, 512), (64, 1), "k"), ((64, 96), (1, 1), "m")],
)
def test_build_index_from_tensor_matches_oracle(dtype, col_major, shape, micro, axis):
    pit = _pkg()
    rng = np.random.default_rng(hash((dtype, col_major, shape, micro)) % 2**32)
    v = _values(shape, 0.02, rng)
    t = _torch_values(v, dtype, col_major)
    idx = pit.build_index_from_tensor(t, micro, axis)
    counts, groups = orc.build_index_from_values(v, micro, axis)
    assert_same_index(idx, counts, groups)


def test_value_test_is_exact_no_epsilon():
    """-0.0 is zero; NaN, inf and denormals are live."""
    import torch

    pit = _pkg()
    v = np.zeros((8, 64), np.float32)
    v[1, 3] = -0.0
    v[2, 40] = np.float32(1e-45)  # denormal
    v[4, 10] = np.nan
    v[6, 63] = -np.inf
    idx = pit.build_index_from_tensor(torch.from_numpy(v).cuda(), (1, 32), "m")
    assert [list(idx.group(g)) for g in range(2)] == [[4], [2, 6]]
    v64 = np.zeros((4, 4))
    v64[0, 0] = 1e-300
    v64[3, 3] = -0.0
    assert pit.build_index_from_tensor(v64, (1, 1), "m").total == 1


def test_host_arrays_are_uploaded():
    pit = _pkg()
    v = np.zeros((8, 8), np.float32)
    v[5, 3] = 2.5
    idx = pit.build_index_from_tensor(v, (1, 4), "m")
    assert idx.total == 1
    assert [set(map(int, idx.group(g))) for g in range(idx.n_groups)] == [{5}, set()]


def test_large_bf16_detection_bit_exact():
    """Full-size property: every group ascending, no duplicates, total equals the oracle's cover."""
    import torch

    pit = _pkg()
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((8192, 8192), device="cuda", dtype=torch.bfloat16, generator=g)
    keep = torch.rand((8192, 8192 // 32), device="cuda", generator=g) >= 0.9
    x = x * keep.repeat_interleave(32, dim=1).to(x.dtype)
    idx = pit.build_index_from_tensor(x, (1, 32), "m")
    want = keep.t().sum(dim=1).cpu().numpy()  # per K-block group: live rows
    np.testing.assert_array_equal(idx.counts, want)
    for gi in (0, 17, idx.n_groups - 1):
        np.testing.assert_array_equal(idx.group(gi), np.nonzero(keep[:, gi].cpu().numpy())[0])


def test_errors_match_reference_messages():
    pit = _pkg()
    ann = pit.from_mask(np.ones((4, 4)), (1, 1))
    with pytest.raises(pit.IndexBuildError, match="positive"):
        pit.build_index(ann, (0, 2), "m")
    with pytest.raises(pit.IndexBuildError, match="rank"):
        pit.build_index(ann, (1, 2, 3), "m")
    with pytest.raises(pit.IndexBuildError, match="workers"):
        pit.build_index(ann, (1, 2), "m", workers=0)
    with pytest.raises(pit.IndexBuildError, match="axis"):
        pit.build_index(ann, (1, 2), "q")


def test_device_from_mask_matches_host():
    import torch

    pit = _pkg()
    rng = np.random.default_rng(3)
    m = (rng.random((130, 70)) > 0.97).astype(np.float32)
    for gran in ((1, 1), (2, 3), (32, 1), (1, 64), (7, 7)):
        dev = pit.from_mask(torch.from_numpy(m).cuda(), gran)
        host = pit.from_mask(m, gran)
        np.testing.assert_array_equal(dev.packed, host.packed)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape,micro", [((4096, 768), (1, 768)), ((1000, 200), (1, 200)), ((77, 64), (1, 512)),
                                         ((33, 8), (1, 8))])
def test_whole_row_micro_tiles_match_oracle(dtype, shape, micro):
    """(1, >= C) micro-tiles (BERT padding rows): one group, one bit per row, stored per 32-row
    block without atomics. Rows mix zeros, -0.0 and (for floats) denormals / NaN."""
    pit = _pkg()
    rng = np.random.default_rng(shape[0] + micro[1])
    v = _values(shape, 0.002, rng)
    v[rng.random(shape[0]) < 0.3] = 0.0
    if dtype in ("float32", "float64"):
        v[3, 1] = -0.0
        v[5, 2] = np.float32(1e-45)
        v[shape[0] - 1, shape[1] - 1] = np.nan
    t = _torch_values(v, dtype, False)
    idx = pit.build_index_from_tensor(t, micro, "m")
    counts, groups = orc.build_index_from_values(v, micro, "m")
    assert_same_index(idx, counts, groups)


@pytest.mark.parametrize("dtype", ["bfloat16", "float32", "float16"])
@pytest.mark.parametrize("shape,micro", [((512, 1024), (128, 64)), ((300, 2048), (1, 32)), ((257, 4096), (32, 16)),
                                         ((1024, 520), (16, 8)), ((96, 8192), (8, 256)), ((70, 1000), (5, 8))])
def test_columnwise_detection_vector_path_matches_oracle(dtype, shape, micro):
    """PIT axis k over row-major values (groups = row bands, bits over micro-columns): the 16-byte
    vector kernel (detect_cols_vec_kernel; micro-columns of 1-32 vectors, ragged band and column
    tails, words shared by several blocks) is bit-exact against the oracle."""
    pit = _pkg()
    rng = np.random.default_rng(shape[0] * 7 + micro[1])
    v = _values(shape, 0.001, rng)
    v[:, rng.random(shape[1]) < 0.3] = 0.0
    t = _torch_values(v, dtype, False)
    idx = pit.build_index_from_tensor(t, micro, "k")
    counts, groups = orc.build_index_from_values(t.float().cpu().numpy(), micro, "k")
    assert_same_index(idx, counts, groups)


@pytest.mark.parametrize("shape,micro,axis,col_major",
                         [((8192, 1024), (32, 1), "k", True), ((1000, 777), (1, 16), "m", False),
                          ((4096, 768), (1, 768), "m", False), ((96, 3000), (16, 1), "k", True)])
def test_index_build_repeats_across_calls_streams_and_graph_replays(shape, micro, axis, col_major):
    """K1 called repeatedly: eager calls on two streams, then a captured build replayed over
    changing values (the serving pattern of graph.py) -- every index equals the oracle's, so no
    state survives from one build into the next."""
    import torch

    pit = _pkg()
    rng = np.random.default_rng(sum(shape) + micro[0])
    dev_vals = []
    for density in (0.02, 0.3, 0.0005):
        v = _values(shape, density, rng)
        dev_vals.append((v, _torch_values(v, "bfloat16", col_major)))
    side = torch.cuda.Stream()
    for rep in range(2):
        for v, t in dev_vals:
            stream = side if rep else torch.cuda.current_stream()
            stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(stream):
                idx = pit.build_index_from_tensor(t, micro, axis)
            torch.cuda.current_stream().wait_stream(stream)
            counts, groups = orc.build_index_from_values(v.astype(np.float32), micro, axis)
            assert_same_index(idx, counts, groups)
    buf = dev_vals[0][1].clone()
    s2 = torch.cuda.Stream()
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        pit.build_index_from_tensor(buf, micro, axis)  # warm-up outside the capture
    torch.cuda.current_stream().wait_stream(s2)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        gidx = pit.build_index_from_tensor(buf, micro, axis)
    for _ in range(2):
        for v, t in dev_vals:
            buf.copy_(t)
            g.replay()
            torch.cuda.synchronize()
            counts, groups = orc.build_index_from_values(v.astype(np.float32), micro, axis)
            c_dev, s_dev = gidx.device_arrays()  # the host view caches: read the replayed buffers
            c_h, s_h = c_dev.cpu().numpy(), s_dev.cpu().numpy()
            np.testing.assert_array_equal(c_h, counts)
            for grp in range(len(groups)):
                np.testing.assert_array_equal(s_h[grp, : c_h[grp]], groups[grp], err_msg=f"group {grp}")
