"""Output-sparse matmul (SDDMM) on the GPU vs the oracle (oracle/pit_oracle.sddmm).

Live micro-tiles of C within the bf16 gate (1e-2 normwise against the f64 product of the
bf16-rounded operands); dead micro-tiles never written (a NaN sentinel survives); the optional
ReLU gate zeroes exactly where gate <= 0; the layout contract raises LayoutError; one CUDA graph
replays equal to the eager call; C3-shaped batched attention scores at full size."""

import numpy as np
import pytest

from oracle import pit_oracle as orc

pytestmark = pytest.mark.gpu


def _bf16(a):
    import torch

    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16)


def _case(M, N, K, gran, zero, seed):
    import torch

    import paper_2301_10936_b200 as pit

    rng = np.random.default_rng(seed)
    A = _bf16(rng.standard_normal((M, K))).cuda()
    Bt = _bf16(rng.standard_normal((N, K))).cuda()  # B column-major = B^T row-major
    ann = pit.random_annotation((M, N), gran, zero, seed=seed)
    return A, Bt, ann


def _check(out, A, Bt, ann, sentinel, gate=None):
    got = out.float().cpu().numpy()
    ref, live = orc.sddmm(A.float().cpu().numpy(), Bt.float().cpu().numpy().T, (ann.tensor_shape, ann.granularity,
                                                                                ann.packed),
                          np.full(got.shape, np.nan), gate=None if gate is None else gate.float().cpu().numpy())
    assert np.isnan(got[~live]).all() if sentinel else (got[~live] == 0).all()
    if live.any():
        assert orc.max_rel_error(got[live], ref[live]) <= 1e-2
    return got, ref, live


@pytest.mark.parametrize("M,N,K,gran,zero", [
    (256, 256, 64, (32, 64), 0.8), (384, 512, 64, (32, 64), 0.5), (1000, 1024, 64, (32, 64), 0.9),
    (512, 768, 128, (1, 32), 0.9), (300, 200, 96, (16, 8), 0.7), (256, 1024, 256, (128, 64), 0.6),
    (128, 320, 72, (64, 128), 0.3), (640, 640, 64, (32, 64), 0.0), (256, 256, 64, (32, 64), 1.0),
    (77, 64, 16, (1, 8), 0.5)])
def test_sddmm_matches_oracle(M, N, K, gran, zero):
    import torch

    from paper_2301_10936_b200.sddmm import run_sddmm

    A, Bt, ann = _case(M, N, K, gran, zero, seed=M + N + K)
    out = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    run_sddmm(A, Bt.t(), ann, out=out)
    torch.cuda.synchronize()
    _check(out, A, Bt, ann, sentinel=True)
    # default out: zeros outside the live micro-tiles (the masked product)
    C = run_sddmm(A, Bt.t(), ann).array
    _check(C, A, Bt, ann, sentinel=False)


def test_sddmm_relu_gate_and_device_annotation():
    import torch

    import paper_2301_10936_b200 as pit
    from paper_2301_10936_b200.sddmm import run_sddmm

    # ReLU-masked activation gradient: dH = (dY . W2^T) * 1[H > 0] inside H's 1x32 micro-tiles
    T, F, D = 512, 1024, 256
    rng = np.random.default_rng(4)
    dY = _bf16(rng.standard_normal((T, D))).cuda()
    W2 = _bf16(rng.standard_normal((F, D)) / 16).cuda()  # [d_ff, d_model]: dH = dY . W2^T, B = W2^T col-major
    keep = rng.random((T, F // 32)) >= 0.9
    H = _bf16(np.maximum(rng.standard_normal((T, F)), 0) * np.repeat(keep, 32, axis=1)).cuda()
    ann = pit.from_mask(H.float().cpu().numpy() != 0, (1, 32)).on_device(torch.device("cuda"))
    out = torch.full((T, F), float("nan"), dtype=torch.bfloat16, device="cuda")
    run_sddmm(dY, W2.t(), ann, out=out, gate=H)
    torch.cuda.synchronize()
    host_ann = pit.from_mask(H.float().cpu().numpy() != 0, (1, 32))
    got, ref, live = _check(out, dY, W2, host_ann, sentinel=True, gate=H)
    h = H.float().cpu().numpy()
    assert (got[live & (h <= 0)] == 0).all()


def test_sddmm_layout_and_shape_errors():
    import torch

    import paper_2301_10936_b200 as pit
    from paper_2301_10936_b200.sddmm import run_sddmm

    A, Bt, ann = _case(256, 256, 64, (32, 64), 0.5, seed=1)
    with pytest.raises(pit.LayoutError, match="col_major"):
        run_sddmm(A, Bt.t().contiguous(), ann)
    with pytest.raises(pit.LayoutError, match="row_major"):
        run_sddmm(A.t().contiguous().t(), Bt.t(), ann)
    with pytest.raises(pit.ExecError, match="annotation"):
        run_sddmm(A, Bt.t(), pit.random_annotation((256, 128), (32, 64), 0.5, seed=1))
    with pytest.raises(pit.ExecError, match="shape"):
        run_sddmm(A[:, :32], Bt.t(), ann)


def test_sddmm_cuda_graph_replay():
    import torch

    from paper_2301_10936_b200.sddmm import output_indexes, run_sddmm

    A, Bt, ann = _case(1024, 1024, 64, (32, 64), 0.8, seed=7)
    ann_d = ann.on_device(torch.device("cuda"))
    eager = run_sddmm(A, Bt.t(), ann_d).array.clone()
    out = torch.zeros_like(eager)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run_sddmm(A, Bt.t(), ann_d, out=out)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run_sddmm(A, Bt.t(), ann_d, out=out, indexes=output_indexes(ann_d))
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)


@pytest.mark.parametrize("heads,seq", [(2, 512), (12, 4096)])
def test_batched_attention_scores(heads, seq):
    """C3 producer side: S = Q . K^T per head inside the Longformer-style 32x64 block mask, all heads
    in one launch; full C3 size (12 heads x 4096^2, head dim 64) against a torch f64 product on the
    device (the oracle's k-loop is too slow at that size; same definition)."""
    import torch

    import paper_2301_10936_b200 as pit
    from paper_2301_10936_b200.sddmm import run_batched_sddmm

    hd = 64
    rng = np.random.default_rng(3)
    qi = np.arange(seq // 32)[:, None] * 32 + 16
    kj = np.arange(seq // 64)[None, :] * 64 + 32
    base = np.abs(qi - kj) <= 256 + 48
    base[:, 0] = True
    base[0, :] = True
    blocks = np.stack([base | (rng.random(base.shape) < 0.02) for _ in range(heads)])
    ann = pit.from_bits(blocks.reshape(heads * seq // 32, seq // 64), (heads * seq, seq), (32, 64))
    g = torch.Generator(device="cuda").manual_seed(5)
    Q = torch.randn((heads, seq, hd), device="cuda", dtype=torch.bfloat16, generator=g)
    Kt = torch.randn((heads, seq, hd), device="cuda", dtype=torch.bfloat16, generator=g)
    out = torch.full((heads, seq, seq), float("nan"), dtype=torch.bfloat16, device="cuda")
    run_batched_sddmm(Q, Kt.transpose(1, 2), ann.on_device(torch.device("cuda")), out=out)
    torch.cuda.synchronize()
    live = torch.from_numpy(blocks).cuda().repeat_interleave(32, 1).repeat_interleave(64, 2)
    assert torch.isnan(out[~live]).all()
    for h in range(heads):
        ref = Q[h].double() @ Kt[h].double().t()
        m = live[h]
        err = float((out[h].double()[m] - ref[m]).abs().max() / ref[m].abs().max())
        assert err <= 1e-2, (h, err)


def test_sddmm_like_detects_the_output_mask_on_device_and_captures():
    """dH = (dY . W2^T) * 1[H > 0] with the output indexes detected from H on the device: equal to the
    annotation-driven call, and a CUDA-graph replay after H changes equals the eager call."""
    import torch

    import paper_2301_10936_b200 as pit
    from paper_2301_10936_b200.sddmm import run_sddmm, run_sddmm_like

    T, F, D = 1024, 2048, 256
    rng = np.random.default_rng(8)
    dY = _bf16(rng.standard_normal((T, D))).cuda()
    W2 = _bf16(rng.standard_normal((F, D)) / 16).cuda()

    def relu_masked(seed):
        r = np.random.default_rng(seed)
        keep = r.random((T, F // 32)) >= 0.95
        return _bf16(np.maximum(r.standard_normal((T, F)), 0) * np.repeat(keep, 32, axis=1)).cuda()

    H = relu_masked(1)
    got = run_sddmm_like(dY, W2.t(), H, (1, 32), gate=H).array
    ann = pit.from_mask(H.float().cpu().numpy() != 0, (1, 32)).on_device(torch.device("cuda"))
    want = run_sddmm(dY, W2.t(), ann, gate=H).array
    assert torch.equal(got, want)
    out = torch.zeros_like(H)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        run_sddmm_like(dY, W2.t(), H, (1, 32), out=out, gate=H)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run_sddmm_like(dY, W2.t(), H, (1, 32), out=out, gate=H)
    H.copy_(relu_masked(2))
    out.zero_()
    g.replay()
    eager = run_sddmm_like(dY, W2.t(), H, (1, 32), gate=H).array
    assert torch.equal(out, eager)
