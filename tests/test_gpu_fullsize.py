"""Parity at BASELINE.json's full sizes through size-independent properties (the f64 oracle is too
slow at 8192^3): the tcgen05 products of the benchmarked configurations must equal cuBLAS on the
operand with every dead micro-tile zeroed (normwise, the bf16 gate), the online index must count
exactly the live micro-tiles of the operand, and dead groups must be exact zeros."""

import pytest

pytestmark = pytest.mark.gpu
BF16_TOL = 1e-2
SIDE = 8192


def _pit():
    import paper_2301_10936_b200 as pit

    return pit


def _plan(t0, axis, tile):
    pit = _pit()
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, "full"))
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=SIDE, k=SIDE, n=SIDE))
    return pit.forced_plan(expr, axis, reg, tile_shape=tile)


def _normwise(x, y):
    return float((x.float() - y.float()).abs().max() / y.float().abs().max().clamp_min(1e-6))


@pytest.mark.parametrize("t0", [32, 128, 256])
def test_pit_k_full_size_matches_cublas_on_masked_operand(t0):
    """C1's distribution (random (t0,1) micro-tiles, 90% zero) at 8192^3: spmm_gk (t0 <= 128) and the
    CTA-pair spmm_gk2 (t0 = 256) against torch.matmul of the same masked bf16 operand."""
    import torch

    pit = _pit()
    g = torch.Generator(device="cuda").manual_seed(t0)
    keep = torch.rand((SIDE, SIDE // t0), device="cuda", generator=g) >= 0.9  # [k, m-block]
    At = torch.randn((SIDE, SIDE), device="cuda", dtype=torch.bfloat16, generator=g)  # A^T [k, m]
    At.mul_(keep.repeat_interleave(t0, dim=1).to(torch.bfloat16))
    A = At.t()  # column-major A [m, k]
    B = torch.randn((SIDE, SIDE), device="cuda", dtype=torch.bfloat16, generator=g)
    plan = _plan(t0, "k", (t0, 64, 256))
    idx = pit.build_index_from_tensor(A, (t0, 1), "k")
    # every kept micro-tile holds Gaussian values, so the index counts exactly the kept ones
    assert idx.total == int(keep.sum().item())
    counts = torch.tensor(list(idx.counts), device="cuda")
    assert torch.equal(counts.to(torch.int64), keep.sum(0).to(torch.int64))
    C = pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx).array
    ref = torch.matmul(A, B)
    assert _normwise(C, ref) <= BF16_TOL
    dead = (keep.sum(0) == 0).nonzero().flatten().tolist()
    for gi in dead[:8]:
        assert torch.count_nonzero(C[gi * t0:(gi + 1) * t0]) == 0


def test_dense_full_size_cta_pairs_match_cublas():
    """The dense plan at 8192^3 runs rowgemm2 (CTA pairs, banded raster) — equal to cuBLAS."""
    import torch

    pit = _pit()
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn((SIDE, SIDE), device="cuda", dtype=torch.bfloat16, generator=g)
    B = torch.randn((SIDE, SIDE), device="cuda", dtype=torch.bfloat16, generator=g)
    plan = _plan(128, "dense", (128, 64, 256))
    C = pit.run_sparse_matmul(plan, pit.DenseTensor(A), pit.DenseTensor(B), None).array
    assert _normwise(C, torch.matmul(A, B)) <= BF16_TOL


# ------------------------------------------------------------------ C3: all heads, full size
def _longformer_blocks(heads, seq, rng, window=256, rand=0.02):
    """Same C3 mask as bench.py: (32 query x 64 key) blocks, sliding window +-256, global first key
    block column and first query block row, plus 2% seeded random blocks per head."""
    import numpy as np

    qi = np.arange(seq // 32)[:, None] * 32 + 16
    kj = np.arange(seq // 64)[None, :] * 64 + 32
    base = np.abs(qi - kj) <= window + 48
    base[:, 0] = True
    base[0, :] = True
    return np.stack([base | (rng.random(base.shape) < rand) for _ in range(heads)])


@pytest.fixture(scope="module")
def c3_operands():
    import numpy as np
    import torch

    heads, seq, hd = 12, 4096, 64
    blocks = _longformer_blocks(heads, seq, np.random.default_rng(3))
    g = torch.Generator(device="cuda").manual_seed(5)
    emask = torch.from_numpy(blocks).cuda().repeat_interleave(32, 1).repeat_interleave(64, 2)
    P = torch.randn((heads, seq, seq), device="cuda", dtype=torch.bfloat16, generator=g)
    P.mul_(emask.to(torch.bfloat16))
    del emask
    V = torch.randn((heads, seq, hd), device="cuda", dtype=torch.bfloat16, generator=g)
    ref = torch.bmm(P.double(), V.double())  # f64 on the same bf16 operands
    return blocks, P, V, ref


@pytest.mark.parametrize("variant", ["k32", "k128", "m64"])
def test_c3_attention_all_heads_full_size(c3_operands, variant):
    """C3 at its full configuration (12 heads x 4096^2 x 64, 32x64 blocks, one batched launch):
    every head within the bf16 gate of the f64 product, for each plan the bench times; the stacked
    index from the device-resident mask equals the one detected from P's values, and the CPU oracle's
    index for the first and last head."""
    import numpy as np
    import torch

    from oracle import pit_oracle as orc

    pit = _pit()
    blocks, P, V, ref = c3_operands
    heads, seq, hd = P.shape[0], P.shape[1], V.shape[2]
    micro, axis, tile = {"k32": ((32, 1), "k", (32, 64, 32)), "k128": ((128, 1), "k", (128, 64, 256)),
                         "m64": ((1, 64), "m", (128, 64, 256))}[variant]
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, "c3"))
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=seq, k=seq, n=hd))
    plan = pit.forced_plan(expr, axis, reg, tile_shape=tile)
    ann = pit.from_bits(blocks.reshape(heads * seq // 32, seq // 64), (heads * seq, seq), (32, 64))
    A3 = P if axis == "m" else pit.stack_slices(P, plan)
    idx = pit.build_index(ann.on_device(), micro, axis)
    O = pit.run_batched_matmul_with_index(plan, A3, V, idx)
    for h in range(heads):
        err = float((O[h].double() - ref[h]).abs().max() / ref[h].abs().max())
        assert err <= BF16_TOL, (h, err)
    if axis == "k":
        idx_v = pit.build_batched_index_from_tensor(A3, micro, "k")
        assert pit.dump_index(idx_v) == pit.dump_index(idx)
        per = seq // micro[0]
        for h in (0, heads - 1):
            a = pit.from_bits(blocks[h], (seq, seq), (32, 64))
            counts, groups = orc.build_index(a.tensor_shape, a.granularity, a.packed, micro, "k")
            assert np.array_equal(idx.counts[h * per:(h + 1) * per], counts)
            for gi in range(0, per, 7):
                assert np.array_equal(idx.group(h * per + gi), groups[gi])
    del A3


# --------------------------------------------------------------- C4: OPT FFN2, full size
@pytest.mark.parametrize("zero", [0.9, 0.99])
def test_c4_opt_ffn2_full_size(zero):
    """C4 at full size (4096 tokens x d_ff 8192 -> d_model 2048, ReLU activations with random 1x32
    micro-tile sparsity): forward pit:m (1,32) and weight-gradient pit:k (32,1) from ONE detection,
    both within the bf16 gate of the f64 products; token rows with no live activation are exact
    zeros; the device index equals the CPU oracle's."""
    import numpy as np
    import torch

    from oracle import pit_oracle as orc

    pit = _pit()
    tokens, d_ff, d_model = 4096, 8192, 2048
    g = torch.Generator(device="cuda").manual_seed(11)
    keep = torch.rand((tokens, d_ff // 32), device="cuda", generator=g) >= zero
    H = torch.relu(torch.randn((tokens, d_ff), device="cuda", dtype=torch.bfloat16, generator=g)) + 0.01
    H = (H * keep.repeat_interleave(32, dim=1).to(torch.bfloat16)).contiguous()
    W2 = torch.randn((d_ff, d_model), device="cuda", dtype=torch.bfloat16, generator=g) * 0.02
    dY = torch.randn((tokens, d_model), device="cuda", dtype=torch.bfloat16, generator=g)
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    fwd = pit.forced_plan(pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"),
                                           dict(m=tokens, k=d_ff, n=d_model)), "m", reg, tile_shape=(16, 32, 128))
    bwd = pit.forced_plan(pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"),
                                           dict(m=d_ff, k=tokens, n=d_model)), "k", reg, tile_shape=(32, 64, 32))
    idx = pit.build_index_from_tensor(H, (1, 32), "m")
    Y = pit.run_matmul_with_index(fwd, pit.DenseTensor(H), pit.DenseTensor(W2), idx).array
    dW2 = pit.run_matmul_with_index(bwd, pit.DenseTensor(H.t()), pit.DenseTensor(dY), idx.transposed()).array
    ry = H.double() @ W2.double()
    rw = H.t().double() @ dY.double()
    assert _normwise(Y, ry) <= BF16_TOL
    assert _normwise(dW2, rw) <= BF16_TOL
    dead_rows = (keep.sum(1) == 0).nonzero().flatten()
    if dead_rows.numel():
        assert torch.count_nonzero(Y[dead_rows]) == 0
    dead_neurons = (keep.sum(0) == 0).nonzero().flatten()
    for nb in dead_neurons[:8].tolist():
        assert torch.count_nonzero(dW2[nb * 32:(nb + 1) * 32]) == 0
    kb = keep.cpu().numpy()
    ann = pit.from_bits(kb, (tokens, d_ff), (1, 32))
    counts, groups = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, (1, 32), "m")
    assert np.array_equal(idx.counts, counts)
    for gi in range(0, idx.n_groups, 17):
        assert np.array_equal(idx.group(gi), groups[gi])
