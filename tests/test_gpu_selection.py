"""GPU: the B200 cost table (profile) and single-tile execution (run_tile, reference tiles.py:119-148)."""

import numpy as np
import pytest

import paper_2301_10936_b200 as pit

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def registry():
    return pit.register_builtin_kernels(include_b200_tiles=True)


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


def test_device_cover_counts_match_reference_golden_and_host():
    import json
    from pathlib import Path

    from paper_2301_10936_b200.index import cover_counts_device
    from paper_2301_10936_b200.policy import cover_group_counts

    cases = json.loads((Path(__file__).parent / "golden" / "index_cases.json").read_text())
    for c in cases:
        ann = pit.random_annotation(c["shape"], c["granularity"], c["zero_ratio"], seed=c["seed"])
        dim = 0 if c["axis"] == "m" else 1
        cands = [(tuple(c["micro"]), dim), ((1, 1), 0), ((3, 5), 1), (tuple(c["micro"]), 1 - dim)]
        got = cover_counts_device(ann, cands)
        assert got[0].tolist() == c["counts"]  # reference build_index counts
        for (m, d), g in zip(cands, got):
            assert g.tolist() == cover_group_counts(ann, m, d).tolist()


def test_selection_device_and_host_candidates_identical(registry):
    from paper_2301_10936_b200.policy import _SampleCovers

    fp = pit.flop_proportional_profile(registry)
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=1024, k=768, n=512))
    samples = [pit.random_annotation((1024, 768), (8, 1), 0.9, seed=s) for s in range(3)]
    keys = [((8, 1), 1), ((1, 32), 0), ((128, 1), 1), ((1, 64), 0)]
    dev = _SampleCovers(samples, keys, device=True)
    host = _SampleCovers(samples, keys, device=False)
    for m, d in keys:
        assert [x.tolist() for x in dev.counts(m, d)] == [x.tolist() for x in host.counts(m, d)]
    cands = pit.selection_candidates(expr, samples, registry, fp)
    assert cands[0].plan == pit.kernel_selection(expr, samples, registry, fp)
