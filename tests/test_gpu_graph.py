"""CUDA-graph replays of the public calls (paper_2301_10936_b200.graph, the bench's timed steps) must
compute exactly what the eager calls compute: detection + SpMM re-run on the current buffer
contents every replay. Covers the gathered-K, split-unit, masked pit:m and single-group paths."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pit():
    import paper_2301_10936_b200 as pit

    return pit


@pytest.mark.parametrize("case", ["pitk_32", "pitk_split", "pitm_masked_pairs", "pitm_masked_single", "pitm_bert"])
def test_graph_replay_equals_eager_and_tracks_new_values(case):
    import torch

    pit = _pit()
    from paper_2301_10936_b200.graph import CapturedSparseMatmul

    rng = np.random.default_rng(hash(case) % 2**32)
    if case == "pitk_32":
        m, k, n, micro, axis, tile = 1024, 2048, 512, (32, 1), "k", (32, 64, 32)
        mask = np.repeat(rng.random((m // 32, k)) >= 0.9, 32, axis=0)
    elif case == "pitk_split":
        m, k, n, micro, axis, tile = 1024, 4096, 64, (128, 1), "k", (128, 64, 256)
        mask = np.repeat(rng.random((m // 128, k)) >= 0.9, 128, axis=0)
        mask[:128] = True
    elif case.startswith("pitm_masked"):
        n = 512 if case.endswith("pairs") else 128
        m, k, micro, axis, tile = 1024, 2048, (1, 32), "m", (128, 32, 256)
        mask = np.repeat(rng.random((m, k // 32)) >= 0.9, 32, axis=1)
    else:
        m, k, n, micro, axis, tile = 2048, 768, 1024, (1, 768), "m", (128, 768, 256)
        mask = np.repeat((rng.random(m) >= 0.4)[:, None], k, axis=1)
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    if reg.get("matmul", tile) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile, "graph"))
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))
    plan = pit.forced_plan(expr, axis, reg, tile_shape=tile)
    A = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float32) * mask).to(torch.bfloat16).cuda()
    if axis == "k":
        A = A.t().contiguous().t()
    B = torch.from_numpy(rng.standard_normal((k, n)).astype(np.float32)).to(torch.bfloat16).cuda()

    def eager():
        idx = pit.build_index_from_tensor(A, micro, axis)
        return pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx).array.clone()

    cap = CapturedSparseMatmul(plan, A, B)
    for _ in range(2):
        out = cap.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager())
    # new values in the same buffers (a different sparsity pattern): the replay re-detects
    A.mul_(torch.from_numpy(rng.random(mask.shape) >= 0.5).to(torch.bfloat16).cuda())
    out = cap.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager())
