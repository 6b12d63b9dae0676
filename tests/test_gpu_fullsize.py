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
    reg = pit.register_builtin_kernels()
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
