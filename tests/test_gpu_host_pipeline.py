"""Host-buffer operands through the public API (the reference's own contract is numpy in, numpy out):
large numpy / pageable B take one pinned copy and the pipelined slab path (B slab uploads, per-slab
SpMM, C slab downloads on three streams). Results equal the device-resident call bitwise."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_numpy_operands_pipelined_equal_device_path(dtype):
    import torch

    import paper_2301_10936_b200 as pit

    m, k, n = 1024, 4096, 4096  # B = 64-128 MiB: over the pipelining threshold
    reg = pit.register_builtin_kernels()
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))
    plan = pit.forced_plan(expr, "k", reg, tile_shape=(32, 64, 32))
    ann = pit.random_annotation((m, k), (32, 1), 0.9, seed=3)
    rng = np.random.default_rng(1)
    A = (rng.standard_normal((m, k)) * ann.materialize(np.float64)).astype(dtype)
    B = rng.standard_normal((k, n)).astype(dtype)
    At = pit.DenseTensor.from_array(A, layout="col_major")
    got = pit.run_sparse_matmul(plan, At, pit.DenseTensor.from_array(B), ann).array
    assert isinstance(got, np.ndarray) and got.dtype == dtype and got.shape == (m, n)
    Ad = torch.from_numpy(np.asfortranarray(A).T.copy()).cuda().t()
    Bd = torch.from_numpy(B).cuda()
    want = pit.run_sparse_matmul(plan, pit.DenseTensor(Ad), pit.DenseTensor(Bd), ann).array.cpu().numpy()
    assert np.array_equal(got, want)
    # pageable torch CPU operands take the same path and come back as torch tensors
    A_cpu = torch.from_numpy(np.asfortranarray(A).T.copy()).t()  # column-major, pageable
    got_t = pit.run_sparse_matmul(plan, pit.DenseTensor(A_cpu), pit.DenseTensor(torch.from_numpy(B)), ann).array
    assert isinstance(got_t, torch.Tensor) and not got_t.is_cuda
    assert np.array_equal(got_t.numpy(), want)
