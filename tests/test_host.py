"""CPU: host-side contract (expressions, plans, annotations, index bookkeeping) — no device."""

import numpy as np
import pytest

import paper_2301_10936_b200 as pit
from oracle import pit_oracle as orc

MATMUL = "C[m,n] += A[m,k] * B[k,n]"


def bound(m, k, n):
    return pit.bind_extents(pit.parse_expr(MATMUL), dict(m=m, k=k, n=n))


def test_pit_axis_table():
    """test_acceptance.py:199-210 operator table."""
    table = {
        "C[p] += A[p,l]": {"p", "l"},
        "C[p] = A[p] + B[p]": {"p"},
        "C[m,n] += A[m,k] * B[k,n]": {"m", "n", "k"},
        "C[b,m,n] += A[b,m,k] * B[b,k,n]": {"b", "m", "n", "k"},
        "C[n,f,x,y] += A[n,m,x+i,y+j] * B[f,m,i,j]": {"n", "m", "f"},
    }
    for text, want in table.items():
        assert pit.pit_axes(pit.parse_expr(text)) == want


def test_operator_kinds_and_simplify():
    assert pit.operator_kind(pit.parse_expr(MATMUL)) == "matmul"
    assert pit.operator_kind(pit.parse_expr("C[b,m,n] += A[b,m,k] * B[b,k,n]")) == "batch_matmul"
    assert pit.operator_kind(pit.parse_expr("C[p] += A[p,l]")) == "reduce_sum"
    assert pit.operator_kind(pit.parse_expr("C[p] = A[p] + B[p]")) == "vec_add"
    reduced, freedom = pit.simplify(pit.parse_expr("C[e,t,f] += X[e,t,d] * W[e,d,f]"))
    assert freedom == {"e": "independent-per-slice"}
    assert pit.operator_kind(reduced) == "matmul"


@pytest.mark.parametrize("bad,needle", [("C[m,n] += A[m,k] * ", "end"), ("C[m+i] += A[m,i]", "compound"),
                                        ("C[m] += A[k]", "output axis"), ("C[m] ? A[m]", "unexpected")])
def test_parse_errors(bad, needle):
    with pytest.raises(pit.ExprError, match=needle):
        pit.parse_expr(bad)


def test_micro_tiles_and_layouts(registry):
    assert pit.get_micro_tile("matmul", (16, 32, 128), "m") == ((1, 32), "row_major")
    assert pit.get_micro_tile("matmul", (16, 32, 128), "k") == ((16, 1), "col_major")
    assert pit.get_micro_tile("matmul", (128, 64, 256), "k") == ((128, 1), "col_major")
    with pytest.raises(pit.PlanError, match="not on the sparse operand"):
        pit.get_micro_tile("matmul", (16, 32, 128), "n")
    plan = pit.forced_plan(bound(1024, 1024, 1024), "dense", registry, tile_shape=(32, 64, 32))
    assert pit.plan_launches(plan, None) == 32 * 16 * 32


def test_cover_count_equals_oracle_index_total():
    rng = np.random.default_rng(0)
    for trial in range(200):
        shape = (int(rng.integers(2, 48)), int(rng.integers(2, 48)))
        gran = (int(rng.integers(1, 5)), int(rng.integers(1, 5)))
        micro = (int(rng.integers(1, 7)), int(rng.integers(1, 7)))
        axis = "m" if rng.integers(2) else "k"
        ann = pit.random_annotation(shape, gran, float(rng.choice([0.0, 0.3, 0.7, 0.95])), seed=trial)
        counts, _ = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, micro, axis)
        assert pit.cover_count(ann, micro, axis) == int(counts.sum())
        np.testing.assert_array_equal(pit.cover_group_counts(ann, micro, axis), counts)


def test_annotation_round_trips(tmp_path):
    ann = pit.random_annotation((40, 30), (3, 4), 0.5, seed=3)
    path = tmp_path / "a.txt"
    pit.save_annotation(ann, path)
    back = pit.load_annotation(path)
    assert back == pit.SparsityAnnotation(ann.tensor_shape, ann.granularity, back.packed)
    np.testing.assert_array_equal(back.packed, ann.packed)
    m = ann.materialize()
    assert np.array_equal(pit.from_mask(m, (3, 4)).packed, ann.packed)
    rag = pit.from_ragged_lengths([3, 0, 16, 7], (4, 16))
    assert rag.materialize().sum(axis=1).tolist() == [3, 0, 16, 7]
    with pytest.raises(pit.AnnotationError):
        pit.from_ragged_lengths([17], (1, 16))


def test_host_index_bookkeeping_without_device():
    counts = np.array([2, 0], np.int64)
    slots = np.array([[5, 1, 0, 0], [0, 0, 0, 0]], np.int64)
    idx = pit.index_from_arrays((1, 4), "m", counts, slots)
    canon = pit.canonicalize(idx)
    assert list(canon.group(0)) == [1, 5]
    assert pit.dump_index(idx) == "microtile 1 4\npit_axis m\ngroup 0 2: 1 5\ngroup 1 0:\n"
    canon.slots[0, 0] = 7  # canonical copies are writable (the reference tests reorder in place)


def test_tensor_file_round_trip(tmp_path):
    rng = np.random.default_rng(2)
    for layout in ("row_major", "col_major"):
        for dt in (np.float32, np.float64):
            t = pit.DenseTensor.from_array(rng.standard_normal((7, 5)), layout=layout, dtype=dt)
            p = tmp_path / f"t_{layout}_{np.dtype(dt).name}.bin"
            pit.save_tensor(t, p)
            back = pit.load_tensor(p)
            assert back.layout == layout and back.dtype == t.dtype
            np.testing.assert_array_equal(back.array, t.array)
            raw = p.read_bytes()
            assert raw[:4] == b"PITT" and len(raw) == 16 + 2 * 8 + 35 * np.dtype(dt).itemsize


def test_permutation_utilities():
    rng = np.random.default_rng(1)
    p = pit.Permutation("k", rng.permutation(9))
    assert np.array_equal(pit.invert(pit.invert(p)).mapping, p.mapping)
    with pytest.raises(pit.ExecError, match="bijection"):
        pit.Permutation("m", np.array([0, 0, 1]))
    x = rng.standard_normal((6, 2))
    rev = pit.Permutation("m", np.arange(6)[::-1])
    assert np.array_equal(pit.apply_permutation(pit.apply_permutation(x, rev), rev), x)


def test_product_package_never_imports_the_oracle():
    import pathlib

    pkg = pathlib.Path(pit.__file__).parent
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "oracle" not in text.replace("oracle\n", "").split("import")[-1] or "from oracle" not in text, f
        assert "from oracle" not in text and "import oracle" not in text, f


def test_device_ops_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    ann = pit.random_annotation((8, 8), (1, 1), 0.5, seed=0)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pit.build_index(ann, (1, 4), "m")


def test_host_pipeline_slab_schedule_tiles_columns():
    """The B / C column slabs of the pinned-host pipeline (executor._slab_schedule) tile [0, N)
    exactly, in order, with no empty slab, small slabs at both ends for wide N."""
    from paper_2301_10936_b200.executor import _slab_schedule

    for N in (1024, 1500, 2048, 3000, 4096, 5000, 8192, 8200, 16384, 65536):
        sched = _slab_schedule(N)
        assert [j0 for j0, _ in sched] == [sum(w for _, w in sched[:i]) for i in range(len(sched))]
        assert sum(w for _, w in sched) == N and all(w > 0 for _, w in sched)
        if N >= 4096:
            widths = [w for _, w in sched]
            assert widths[0] < max(widths) and widths[-1] < max(widths)
