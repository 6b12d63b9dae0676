"""CPU: files WRITTEN BY THE REFERENCE in its own formats are read by this package, and this
package writes the same bytes back.

tests/golden/wire/ was produced by `pittile` itself (tests/golden/make_golden.py wire_cases /
wire_cli): annotation text (reference sparsity.py:135-167), PITT tensors (executor.py:93-116),
canonical index dumps (index.py:185-195), a `pit-profile v1` cost table (tiles.py:224-270) and a
`pittile bench` CSV (cli.py:330). The GPU replay of the same files is tests/test_gpu_golden.py.
"""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2301_10936_b200 as pit
from oracle import pit_oracle as orc

WIRE = Path(__file__).resolve().parent / "golden" / "wire"
CASES = json.loads((WIRE / "wire_cases.json").read_text())
ANNS = sorted(p.name for p in WIRE.glob("*.ann"))
PITTS = sorted(p.name for p in WIRE.glob("*.pitt"))
REF_CSV_HEADER = "op,shape,granularity,zero_ratio,plan,microtile,tile,launches,wall_ms,dense_wall_ms,speedup"


@pytest.mark.parametrize("name", ANNS)
def test_annotation_text_round_trips_byte_for_byte(name, tmp_path):
    ann = pit.load_annotation(WIRE / name)
    pit.save_annotation(ann, tmp_path / name)
    assert (tmp_path / name).read_bytes() == (WIRE / name).read_bytes()


def test_annotation_text_matches_seeded_generator():
    for c in CASES:
        ann = pit.load_annotation(WIRE / f"{c['name']}.ann")
        gen = pit.random_annotation(tuple(c["shape"][:2]), tuple(c["granularity"]), c["zero_ratio"], seed=c["seed"])
        assert ann.tensor_shape == gen.tensor_shape and np.array_equal(ann.packed, gen.packed), c["name"]
    c1 = pit.load_annotation(WIRE / "c1_1024.ann")
    assert np.array_equal(c1.packed, pit.random_annotation((1024, 1024), (32, 1), 0.9, seed=1).packed)


@pytest.mark.parametrize("name", PITTS)
def test_pitt_tensor_round_trips_byte_for_byte(name, tmp_path):
    t = pit.load_tensor(WIRE / name)
    pit.save_tensor(t, tmp_path / name)
    assert (tmp_path / name).read_bytes() == (WIRE / name).read_bytes()


def test_pitt_layout_flag_is_kept():
    for c in CASES:
        A = pit.load_tensor(WIRE / f"{c['name']}_A.pitt")
        want = "col_major" if c["axis"] == "k" else "row_major"
        assert A.layout == want or min(A.shape) == 1, c["name"]


@pytest.mark.parametrize("c", [c for c in CASES if c["axis"] != "dense"], ids=lambda c: c["name"])
def test_index_dump_files_match_oracle_and_host_dump(c):
    """The reference's dump file is what the oracle (and the host dump of the same index) prints."""
    ann = pit.load_annotation(WIRE / f"{c['name']}.ann")
    counts, groups = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, tuple(c["micro"]), c["axis"])
    text = (WIRE / f"{c['name']}.index").read_text()
    assert orc.dump_index(c["micro"], c["axis"], counts, groups) == text
    pg = max([len(g) for g in groups] + [1])
    slots = np.zeros((len(groups), max(pg, 1)), np.int64)
    for g, coords in enumerate(groups):
        slots[g, : len(coords)] = coords
    host = pit.index_from_arrays(tuple(c["micro"]), c["axis"], counts, slots)
    assert pit.dump_index(host) == text


def test_c1_index_dump_matches_oracle():
    ann = pit.load_annotation(WIRE / "c1_1024.ann")
    counts, groups = orc.build_index(ann.tensor_shape, ann.granularity, ann.packed, (32, 1), "k")
    assert orc.dump_index((32, 1), "k", counts, groups) == (WIRE / "c1_1024.index").read_text()


def test_pitt_results_match_oracle():
    """The reference's C (fp32 tile loop) and R (f64 oracle) files against the CPU oracle."""
    for c in CASES:
        A = pit.load_tensor(WIRE / f"{c['name']}_A.pitt").array
        B = pit.load_tensor(WIRE / f"{c['name']}_B.pitt").array
        R = pit.load_tensor(WIRE / f"{c['name']}_R.pitt").array
        Cref = pit.load_tensor(WIRE / f"{c['name']}_C.pitt").array
        np.testing.assert_array_equal(orc.dense_reference_f64(A, B), R)
        assert orc.verify_close(Cref, R)


def test_reference_profile_file_loads_and_round_trips(tmp_path):
    import warnings

    with warnings.catch_warnings():  # the reference's CPU run may carry another machine's fingerprint
        warnings.simplefilter("ignore")
        table = pit.load_profile(WIRE / "pittile_cpu.prof")
    assert len(table.costs) >= 4
    pit.save_profile(table, tmp_path / "p.prof")
    assert (tmp_path / "p.prof").read_bytes() == (WIRE / "pittile_cpu.prof").read_bytes()


def test_bench_csv_schema_extends_the_reference():
    """bench.py --csv writes the reference's `pittile bench` columns first, then the B200 ones."""
    import bench

    ref_header = (WIRE / "pittile_bench.csv").read_text().splitlines()[0]
    assert ref_header == REF_CSV_HEADER
    cols = bench.CSV_COLUMNS
    assert ",".join(cols[: len(ref_header.split(","))]) == ref_header
    assert cols[len(ref_header.split(",")):] == ["eff_tflops", "gbps", "roofline_frac"]
    rows = bench.read_bench_csv(WIRE / "pittile_bench.csv")
    assert [r["plan"] for r in rows] == ["pit:k", "dense", "pit:k", "dense"]
