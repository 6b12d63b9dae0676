"""fp16 operands on every tensor-core kernel (the north-star gate covers bf16 AND fp16: 1e-2 normwise
against the reference's fp32 result). Same plans as the bf16 suites, one shape each."""

import numpy as np
import pytest

from oracle import pit_oracle as orc

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _pit():
    import paper_2301_10936_b200 as pit

    return pit


def _plan(m, k, n, axis, tile):
    pit = _pit()
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, "fp16"))
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))
    return pit.forced_plan(expr, axis, reg, tile_shape=tile)


@pytest.mark.parametrize("axis,micro,tile", [
    ("k", (32, 1), (32, 64, 256)),     # spmm_gk, orientation T
    ("k", (128, 1), (128, 64, 256)),   # spmm_gk, orientation N
    ("k", (256, 1), (256, 64, 256)),   # spmm_gk2, CTA pairs
    ("m", (1, 64), (128, 64, 256)),    # rowgemm, union rows
    ("m", (1, 32), (128, 32, 256)),    # rowgemm2 masked mode (union ~86% of rows), CTA pairs
    ("dense", None, (128, 64, 256)),   # rowgemm2, CTA pairs
])
def test_fp16_plans_match_oracle(axis, micro, tile):
    import torch

    pit = _pit()
    m, k, n = 512, 384, 520
    plan = _plan(m, k, n, axis, tile)
    rng = np.random.default_rng(7)
    A = rng.standard_normal((m, k)).astype(np.float32)
    ann = None
    if micro is not None:
        ann = pit.random_annotation((m, k), micro, 0.85, seed=3)
        A *= ann.materialize()
    B = rng.standard_normal((k, n)).astype(np.float32)
    At = torch.from_numpy(A).to(torch.float16).cuda()
    if axis == "k":
        At = At.t().contiguous().t()
    Bt = torch.from_numpy(B).to(torch.float16).cuda()
    C = pit.run_sparse_matmul(plan, pit.DenseTensor(At), pit.DenseTensor(Bt), ann).array
    assert C.dtype == torch.float16 and C.is_cuda
    Ar, Br = At.float().cpu().numpy(), Bt.float().cpu().numpy()
    if ann is None:
        ref = orc.dense_reference_f64(Ar, Br)
    else:
        ref = orc.run_sparse_matmul(Ar, Br, (ann.tensor_shape, ann.granularity, ann.packed), axis, tile, np.float64)
    assert orc.max_rel_error(C.float().cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("T,E", [(2000, 16), (3000, 2)])
def test_fp16_moe_layer(T, E):
    """Grouped GEMMs in fp16: small groups (rowgemm2t) and large groups (rowgemm2)."""
    import torch

    from paper_2301_10936_b200.moe import SwitchMoE

    d, F = 128, 256
    rng = np.random.default_rng(T)
    x = rng.standard_normal((T, d)).astype(np.float32)
    logits = rng.standard_normal((T, E)).astype(np.float32)
    w1 = (rng.standard_normal((E, d, F)) / np.sqrt(d)).astype(np.float32)
    w2 = (rng.standard_normal((E, F, d)) / np.sqrt(F)).astype(np.float32)
    h16 = lambda a: torch.from_numpy(a).to(torch.float16).cuda()  # noqa: E731
    layer = SwitchMoE(h16(w1), h16(w2), E)
    out = layer(h16(x), torch.from_numpy(logits).cuda()).float().cpu().numpy()
    r16 = lambda a: torch.from_numpy(a).to(torch.float16).float().numpy()  # noqa: E731
    ref = orc.switch_forward(r16(x), logits, r16(w1), r16(w2),
                             round_hidden=lambda h: torch.from_numpy(h).to(torch.float16).float().numpy())
    assert orc.max_rel_error(out, ref) <= TOL


def test_fp16_split_gathered_k_units():
    """Split units (few, unequal 128-row groups, N <= 64) in fp16: a global group sees every key."""
    import torch

    pit = _pit()
    m, k, n = 1024, 4096, 64
    plan = _plan(m, k, n, "k", (128, 64, 256))
    rng = np.random.default_rng(11)
    mask = np.repeat(rng.random((m // 128, k)) >= 0.9, 128, axis=0)
    mask[:128] = True
    A = rng.standard_normal((m, k)).astype(np.float32) * mask
    B = rng.standard_normal((k, n)).astype(np.float32)
    At = torch.from_numpy(A).to(torch.float16).cuda().t().contiguous().t()
    Bt = torch.from_numpy(B).to(torch.float16).cuda()
    idx = pit.build_index_from_tensor(At, (128, 1), "k")
    C = pit.run_matmul_with_index(plan, pit.DenseTensor(At), pit.DenseTensor(Bt), idx).array
    assert C.dtype == torch.float16
    ref = orc.dense_reference_f64(At.float().cpu().numpy(), Bt.float().cpu().numpy())
    assert orc.max_rel_error(C.float().cpu().numpy(), ref) <= TOL
