"""GPU: the B200 cost table (profile) and single-tile execution (run_tile, reference tiles.py:119-148)."""

import numpy as np
import pytest

import paper_2301_10936_b200 as pit

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def registry():
    return pit.register_builtin_kernels()


@pytest.fixture(scope="module")
def measured(registry):
    return pit.profile(registry, reps=3, warmup=1, reps_inner=3, extent=1024)


def test_profile_covers_registry_with_positive_costs(registry, measured):
    assert len(measured) == len(registry)
    for d in registry:
        assert measured.cost(d) > 0.0
    assert measured.reps == 3 and not measured.foreign


def test_profile_tensor_core_tiles_cheaper_per_flop(registry, measured):
    # the 128-row tiles drive the tcgen05 gather kernel; the 8-row ones a narrow gather
    per_flop = lambda d: measured.cost(d) / d.flops  # noqa: E731
    assert per_flop(registry.get("matmul", (128, 64, 256))) < per_flop(registry.get("matmul", (8, 32, 128)))


def test_measured_selection_is_well_formed(registry, measured, tmp_path):
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=2048, k=2048, n=2048))
    samples = [pit.random_annotation((2048, 2048), (32, 1), 0.95, seed=s) for s in range(2)]
    plan = pit.kernel_selection(expr, samples, registry, measured)
    assert not plan.is_dense
    pit.save_profile(measured, tmp_path / "b200.prof")
    again = pit.kernel_selection(expr, samples, registry, pit.load_profile(tmp_path / "b200.prof"))
    assert (again.tile, again.pit_axis) == (plan.tile, plan.pit_axis)


def test_run_tile_matches_numpy(registry):
    rng = np.random.default_rng(3)
    for d in registry:
        ins_shapes, out_shape = d.buffer_shapes()
        ins = [rng.standard_normal(s).astype(np.float32) for s in ins_shapes]
        out = rng.standard_normal(out_shape).astype(np.float32)
        want = out.astype(np.float64)
        if d.op_kind == "matmul":
            want = want + ins[0].astype(np.float64) @ ins[1].astype(np.float64)
        elif d.op_kind == "reduce_sum":
            want = want + ins[0].astype(np.float64).sum(axis=1)
        else:
            want = ins[0].astype(np.float64) + ins[1]
        pit.run_tile(d, ins, out)
        assert pit.max_rel_error(out, want) <= 1e-5, d


def test_run_tile_device_buffers(registry):
    import torch

    d = registry.get("matmul", (32, 64, 32))
    a = torch.randn(32, 64, device="cuda")
    b = torch.randn(64, 32, device="cuda")
    out = torch.ones(32, 32, device="cuda")
    scratch = torch.empty(32, 32, device="cuda")
    pit.run_tile(d, [a, b], out, scratch)
    ref = 1.0 + a.double() @ b.double()
    assert float((out.double() - ref).abs().max() / ref.abs().max()) <= 1e-5
