"""The pipelined fp32 pit:k kernel (K7b, csrc/pit_spmm_simt.cu) against the generic K7 kernel it
replaces for BASELINE configs[0] (C1: 1024^3 fp32, 32x1 micro-tiles, TF32 never used): bitwise equal
(same fma order: the group's stored k order), and within 1e-5 of the f64 oracle, over ragged shapes."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

CODE = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2301_10936_b200 as pit
m, k, n, t0 = (int(x) for x in sys.argv[2:6])
zero = float(sys.argv[6])
g = torch.Generator(device="cuda").manual_seed(m + k + n)
keep = torch.rand((k, -(-m // t0)), device="cuda", generator=g) >= zero
At = torch.randn((k, m), device="cuda", generator=g) * keep.repeat_interleave(t0, dim=1)[:, :m].float()
A = At.t()
B = torch.randn((k, n), device="cuda", generator=g)
reg = pit.register_builtin_kernels(include_b200_tiles=True)
tile = (t0, 64, 32)
if reg.get("matmul", tile) is None:
    reg.register(pit.TileKernelDescriptor("matmul", tile, "t"))
plan = pit.forced_plan(pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n)), "k", reg, tile_shape=tile)
idx = pit.build_index_from_tensor(A, (t0, 1), "k")
C = pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx).array
ref = A.double() @ B.double()
err = float((C.double() - ref).norm() / ref.norm().clamp_min(1e-30))
np.save(sys.argv[1], C.cpu().numpy())
print(err)
""" % str(ROOT)


@pytest.mark.parametrize("shape", [(1024, 1024, 1024, 32, 0.9), (1000, 777, 516, 32, 0.8), (256, 4096, 128, 64, 0.95),
                                   (96, 300, 4, 8, 0.5)])
def test_pipelined_fp32_pitk_bitwise_equal_to_generic(shape, tmp_path):
    outs = []
    for flag in ("1", "0"):
        f = str(tmp_path / f"c{flag}.npy")
        r = subprocess.run([sys.executable, "-c", CODE, f, *map(str, shape)], env=dict(os.environ, PIT_SIMT_GK=flag),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        assert float(r.stdout.strip().splitlines()[-1]) <= 1e-5
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])
