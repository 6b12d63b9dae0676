"""CPU: pin the oracle (and the host-side API) to the reference's own outputs.

Fixtures in tests/golden/ were produced by running the reference pittile package
(tests/golden/make_golden.py). No GPU needed.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import pit_oracle as orc

GOLD = Path(__file__).resolve().parent / "golden"


def _json(name):
    return json.loads((GOLD / name).read_text())


INDEX_CASES = _json("index_cases.json")


@pytest.mark.parametrize("case", INDEX_CASES, ids=lambda c: f"{c['shape']}-{c['granularity']}-{c['micro']}-{c['axis']}")
def test_oracle_index_matches_reference_dump(case):
    ann = (tuple(case["shape"]), tuple(case["granularity"]), np.array(case["packed"], np.uint8))
    counts, groups = orc.build_index(*ann, tuple(case["micro"]), case["axis"])
    assert counts.tolist() == case["counts"]
    assert orc.dump_index(case["micro"], case["axis"], counts, groups) == case["dump"]
    # ascending == reference workers=1 order
    for g in groups:
        assert np.all(np.diff(g) > 0)


def test_host_annotation_generator_is_bit_identical():
    import paper_2301_10936_b200 as pit

    for case in INDEX_CASES:
        ann = pit.random_annotation(case["shape"], case["granularity"], case["zero_ratio"], seed=case["seed"])
        assert ann.packed.tolist() == case["packed"]
        assert pit.cover_count(ann, case["micro"], case["axis"]) == case["cover"]


def test_oracle_value_route_matches_reference():
    arrays = np.load(GOLD / "value_cases.npz")
    for c in _json("value_cases.json"):
        counts, groups = orc.build_index_from_values(arrays[c["key"]], c["micro"], c["axis"])
        assert orc.dump_index(c["micro"], c["axis"], counts, groups) == c["dump"], c["key"]


def test_oracle_gather_scatter_matches_reference():
    data = np.load(GOLD / "gather_cases.npz")
    meta = _json("gather_cases.json")
    for c in meta["cases"]:
        shape, micro, axis, tshape = meta["specs"][c["case"]]
        src = data[f"src{c['case']}"]
        _, groups = orc.build_index(*orc.mask_to_ann(src, (1, 1)), tuple(micro), axis)
        d = orc.PIT_DIMS[axis]
        tile = np.full(tuple(tshape), 9.0, np.float32)
        n = orc.sread(src, groups, micro, d, c["group"], tile, start=c["start"])
        assert n == c["n"]
        np.testing.assert_array_equal(tile, data[c["key"] + "_tile"])
        dst = np.zeros_like(src)
        orc.swrite(tile, dst, groups, micro, d, c["group"], start=c["start"])
        np.testing.assert_array_equal(dst, data[c["key"] + "_dst"])
        acc = np.ones_like(src)
        orc.swrite(tile, acc, groups, micro, d, c["group"], start=c["start"], accumulate=True)
        np.testing.assert_array_equal(acc, data[c["key"] + "_acc"])


def test_oracle_matmul_matches_reference():
    data = np.load(GOLD / "matmul_cases.npz")
    for c in _json("matmul_cases.json"):
        i = c["i"]
        A, B = data[f"A{i}"], data[f"B{i}"]
        m, k, n = c["shape"]
        ann = ((m, k), tuple(c["granularity"]), np.array(c["packed"], np.uint8))
        C = orc.run_sparse_matmul(A, B, ann, c["axis"], tuple(c["tile"]))
        # same tile algorithm, fp32: equal up to BLAS kernel rounding differences
        assert orc.max_rel_error(C, data[f"C{i}"]) <= 1e-6, i
        # f64 oracle is bit-identical to the reference's run_dense_reference
        np.testing.assert_array_equal(orc.dense_reference_f64(A, B), data[f"R{i}"])
        assert orc.verify_close(data[f"C{i}"], data[f"R{i}"])
        if c["axis"] != "dense":
            M_t, K_t, _ = c["tile"]
            micro = (1, K_t) if c["axis"] == "m" else (M_t, 1)
            counts, _ = orc.build_index(*ann, micro, c["axis"])
            assert orc.plan_launches(counts, c["axis"], c["tile"], n) == c["launches"]
            assert int(counts.sum()) == c["gathered"]


def test_host_plan_contract_matches_reference():
    import paper_2301_10936_b200 as pit

    gold = _json("plan_cases.json")
    for key, (micro, layout) in gold["micro"].items():
        tile, axis = key.split(":")
        got = pit.get_micro_tile("matmul", tuple(int(x) for x in tile.split("x")), axis)
        assert [list(got[0]), got[1]] == [micro, layout]
    reg = pit.register_builtin_kernels()
    for c in gold["launches"]:
        m, k, n = c["shape"]
        expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))
        plan = pit.forced_plan(expr, c["axis"], reg, tile_shape=tuple(c["tile"]))
        ann = pit.random_annotation((m, k), (2, 3), 0.7, seed=c["seed"])
        assert pit.plan_launches(plan, ann if c["axis"] != "dense" else None) == c["launches"]


def test_cover_table_matches_published_search_results():
    """PAPER.md:1072-1094 / test_acceptance.py:44-67: cover-sparsity within 1 pp."""
    import paper_2301_10936_b200 as pit

    published = [66.39, 96.06, 81.45, 96.05, 95.0, 96.02, 95.0, 99.0]
    for row, pub in zip(_json("plan_cases.json")["cover_table"], published):
        ann = pit.random_annotation((4096, 4096), row["granularity"], row["zero_ratio"], seed=row["seed"])
        mt = tuple(row["micro"])
        cov = pit.cover_count(ann, mt, "m")
        assert cov == row["cover"]
        grid = (4096 // mt[0]) * (4096 // mt[1])
        assert abs(100.0 * (1 - cov / grid) - pub) <= 1.0


def test_oracle_reduce_sum_matches_reference():
    data = np.load(GOLD / "reduce_cases.npz")
    for c in _json("reduce_cases.json"):
        i = c["i"]
        ann = (tuple(c["shape"]), (1, 1), np.array(c["packed"], np.uint8))
        got = orc.reduce_sum(data[f"A{i}"], ann, c["axis"], (16, 64))
        assert orc.max_rel_error(got, data[f"C{i}"]) <= 1e-6, i
