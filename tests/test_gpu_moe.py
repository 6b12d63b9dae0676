"""MoE dispatch on the GPU vs the oracle: routing index bit-exact, grouped expert GEMMs and the
gate-scaled combine within the bf16 gate (1e-2 normwise) of the f64 oracle."""

import numpy as np
import pytest

from oracle import pit_oracle as orc

pytestmark = pytest.mark.gpu


def _bf16_round(a):
    import torch

    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def _problem(T, E, d, F, seed, skew=0.0):
    rng = np.random.default_rng(seed)
    x = _bf16_round(rng.standard_normal((T, d)))
    logits = rng.standard_normal((T, E)).astype(np.float32)
    logits[:, 0] += skew  # imbalanced routing
    w1 = _bf16_round(rng.standard_normal((E, d, F)) / np.sqrt(d))
    w2 = _bf16_round(rng.standard_normal((E, F, d)) / np.sqrt(F))
    return x, logits, w1, w2


def _cuda(a, dtype=None):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.to(dtype) if dtype is not None else t


def test_route_index_is_bit_exact():
    import torch

    from paper_2301_10936_b200.moe import CudaBackend

    be = CudaBackend()
    for T, E in ((1, 4), (37, 8), (1000, 128), (4097, 64)):
        rng = np.random.default_rng(T)
        logits = rng.standard_normal((T, E)).astype(np.float32)
        logits[::7, 3] = logits[::7].max(axis=1)  # ties -> lowest expert
        expert, gate, counts, slots = be.route(_cuda(logits))
        oe, og, oc, og_groups = orc.switch_route(logits)
        np.testing.assert_array_equal(expert.cpu().numpy(), oe)
        np.testing.assert_allclose(gate.cpu().numpy(), og, rtol=1e-5)
        np.testing.assert_array_equal(counts.cpu().numpy(), oc)
        sl = slots.cpu().numpy()
        for e in range(E):
            np.testing.assert_array_equal(sl[e, : oc[e]], og_groups[e])
        offsets, tiles, perm = be.plan(counts, slots, slots.shape[1], T)
        np.testing.assert_array_equal(offsets.cpu().numpy(), np.concatenate([[0], np.cumsum(oc)]))
        np.testing.assert_array_equal(perm.cpu().numpy(), np.concatenate(og_groups))


@pytest.mark.parametrize("T,E,d,F,skew", [(1000, 8, 256, 512, 0.0), (4096, 128, 768, 3072, 0.0),
                                          (3000, 16, 128, 256, 3.0), (5, 4, 64, 128, 0.0),
                                          (4100, 4, 192, 320, 1.0), (4096, 4, 256, 384, 0.0)])
def test_switch_layer_single_gpu_matches_oracle(T, E, d, F, skew):
    # small groups (< 256 tokens per expert on average) run the swapped-role rowgemm2t, large ones
    # the 256-row pair tiles of rowgemm2 (the last case: ~1025 tokens per expert, ragged tails)
    import torch

    from paper_2301_10936_b200.moe import SwitchMoE

    x, logits, w1, w2 = _problem(T, E, d, F, seed=T + E, skew=skew)
    layer = SwitchMoE(_cuda(w1, torch.bfloat16), _cuda(w2, torch.bfloat16), E)
    out = layer(_cuda(x, torch.bfloat16), _cuda(logits)).float().cpu().numpy()
    ref = orc.switch_forward(x, logits, w1, w2, round_hidden=_bf16_round)
    assert orc.max_rel_error(out, ref) <= 1e-2


def test_expert_parallel_path_on_one_rank():
    """The all-to-all orchestration with a single-rank NCCL group equals the local path."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2301_10936_b200.moe import SwitchMoE

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        x, logits, w1, w2 = _problem(777, 8, 128, 256, seed=3)
        layer = SwitchMoE(_cuda(w1, torch.bfloat16), _cuda(w2, torch.bfloat16), 8)
        local = layer(_cuda(x, torch.bfloat16), _cuda(logits)).float().cpu().numpy()
        ep = layer._forward_ep(_cuda(x, torch.bfloat16), _cuda(logits)).float().cpu().numpy()
        ref = orc.switch_forward(x, logits, w1, w2, round_hidden=_bf16_round)
        assert orc.max_rel_error(ep, ref) <= 1e-2
        # the EP path applies the gate after the bf16 round trip through the all-to-all
        assert orc.max_rel_error(ep, local) <= 1e-2
    finally:
        dist.destroy_process_group()


def test_grouped_gemm_batched_slices():
    """Per-slice independent PIT plans (prevalent axis, expr.py simplify): a batched gathered-row GEMM
    with arbitrary per-slice row lists equals per-slice dense products."""
    import torch

    from paper_2301_10936_b200.moe import CudaBackend

    be = CudaBackend()
    rng = np.random.default_rng(0)
    G, rows_a, K, N = 6, 500, 192, 320
    A = _bf16_round(rng.standard_normal((rows_a, K)))
    W = _bf16_round(rng.standard_normal((G, K, N)) / np.sqrt(K))
    counts = rng.integers(0, 200, size=G).astype(np.int32)
    src = np.zeros((G, 256), np.int32)
    for g in range(G):
        src[g, : counts[g]] = rng.choice(rows_a, size=counts[g], replace=False)
    ct = _cuda(counts)
    off, tiles, _ = be.plan(ct)
    out = torch.zeros((int(counts.sum()), N), dtype=torch.bfloat16, device="cuda")
    be.grouped_gemm(_cuda(A, torch.bfloat16), _cuda(W, torch.bfloat16), ct, off, tiles, out, row_src=_cuda(src),
                    src_stride=256)
    got = out.float().cpu().numpy()
    o = np.concatenate([[0], np.cumsum(counts)])
    for g in range(G):
        ref = A[src[g, : counts[g]]].astype(np.float64) @ W[g].astype(np.float64)
        if counts[g]:
            assert orc.max_rel_error(got[o[g] : o[g + 1]], ref) <= 1e-2


def test_ffn1_packing_is_bitwise_the_gathered_product():
    """Large expert groups pack FFN1's tokens into expert order first (pit_pack_groups, TMA-fed A):
    the same tiles in the same order as the cp.async row gathers, so bitwise the same layer output
    (PIT_MOE_PACK=1 vs =0 in child processes)."""
    import os
    import subprocess
    import sys
    import tempfile
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2301_10936_b200.moe import SwitchMoE
g = torch.Generator(device="cuda").manual_seed(7)
T, E, d, F = 8192, 16, 512, 1024
x = torch.randn((T, d), device="cuda", generator=g).to(torch.bfloat16)
logits = torch.randn((T, E), device="cuda", generator=g)
w1 = (torch.randn((E, d, F), device="cuda", generator=g) / 24).to(torch.bfloat16)
w2 = (torch.randn((E, F, d), device="cuda", generator=g) / 32).to(torch.bfloat16)
out = SwitchMoE(w1, w2, E)(x, logits)
np.save(sys.argv[1], out.view(torch.int16).cpu().numpy())
""" % str(root)
    outs = []
    for flag in ("1", "0"):
        f = tempfile.mktemp(suffix=".npy")
        r = subprocess.run([sys.executable, "-c", code, f], env=dict(os.environ, PIT_MOE_PACK=flag),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])
