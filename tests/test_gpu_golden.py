"""GPU: replay the REFERENCE's own outputs directly against the CUDA path.

Every fixture here was produced by running `pittile` itself (tests/golden/make_golden.py):
  index_cases.json   71 annotation -> canonical dump_index text (reference index.py:102-195)
  value_cases.*      6 raw-value cases incl. -0.0 / NaN / inf / denormals (index.py:164-173)
  gather_cases.*     SRead / SWrite known answers incl. start offsets, edge zero-fill and accumulate
                     (executor.py:170-264)
  matmul_cases.*     11 fp32 run_sparse_matmul results + the f64 oracle + ExecStats (executor.py:464-537)
  wire/              files the reference wrote in its own formats (annotation text, PITT, index dumps)
The CPU suite pins the oracle to the same fixtures (test_oracle_golden.py, test_wire_formats.py);
here the sm_100a kernels are compared with the reference's recorded results without the oracle in
between. Index parity is bit-exact (equal dump text); fp32 products within 1e-5 normwise of the f64
oracle (TF32 never used) and of the reference's own fp32 result; SRead/SWrite bit-exact.
"""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
WIRE = GOLD / "wire"
FP32_TOL = 1e-5


def _pit():
    import paper_2301_10936_b200 as pit

    return pit


def _json(name):
    return json.loads((GOLD / name).read_text())


INDEX_CASES = _json("index_cases.json")
VALUE_CASES = _json("value_cases.json")
MATMUL_CASES = _json("matmul_cases.json")
GATHER = _json("gather_cases.json")
WIRE_CASES = json.loads((WIRE / "wire_cases.json").read_text())


def _bound(m, k, n):
    pit = _pit()
    return pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=m, k=k, n=n))


# ------------------------------------------------------------------------------ K1 detection
@pytest.mark.parametrize("case", INDEX_CASES, ids=lambda c: f"{c['shape']}-{c['granularity']}-{c['micro']}-{c['axis']}")
def test_gpu_index_equals_reference_dump(case):
    """Annotation route: the device index prints exactly the reference's dump, and its groups come
    back in the reference's workers=1 (ascending) order."""
    pit = _pit()
    ann = pit.SparsityAnnotation(tuple(case["shape"]), tuple(case["granularity"]), np.array(case["packed"], np.uint8))
    idx = pit.build_index(ann, tuple(case["micro"]), case["axis"])
    assert idx.counts.tolist() == case["counts"]
    assert idx.total == case["total"]
    assert pit.dump_index(idx) == case["dump"]
    for g in range(idx.n_groups):
        assert np.all(np.diff(idx.group(g)) > 0)
    # the same bits on the device (capturable route) give the same index
    idx_d = pit.build_index(ann.on_device(), tuple(case["micro"]), case["axis"])
    assert pit.dump_index(idx_d) == case["dump"]


@pytest.mark.parametrize("layout", ["row_major", "col_major"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_gpu_value_route_equals_reference_dump(layout, dtype):
    """Value route (v != 0.0): -0.0 dead, NaN / inf / fp32 denormal live, exactly as the reference."""
    import torch

    pit = _pit()
    arrays = np.load(GOLD / "value_cases.npz")
    for c in VALUE_CASES:
        v = arrays[c["key"]]
        t = torch.from_numpy(v.astype(np.float64) if dtype == "f64" else v).cuda()
        if layout == "col_major":
            t = t.t().contiguous().t()
        idx = pit.build_index_from_tensor(t, tuple(c["micro"]), c["axis"])
        assert pit.dump_index(idx) == c["dump"], c["key"]
    # numpy host input through the reference's call shape
    for c in VALUE_CASES:
        idx = pit.build_index_from_tensor(arrays[c["key"]], tuple(c["micro"]), c["axis"])
        assert pit.dump_index(idx) == c["dump"], c["key"]


# ------------------------------------------------------------------------- K5 SRead / SWrite
def _gather_inputs(c):
    pit = _pit()
    data = np.load(GOLD / "gather_cases.npz")
    shape, micro, axis, tshape = GATHER["specs"][c["case"]]
    src = data[f"src{c['case']}"]
    idx = pit.build_index(pit.from_mask(src, (1, 1)), tuple(micro), axis)
    return data, src, idx, tuple(tshape)


@pytest.mark.parametrize("c", GATHER["cases"], ids=lambda c: c["key"])
def test_gpu_sread_swrite_equal_reference_known_answers(c):
    """numpy in / numpy out (the reference's contract): tile, assigned dst and accumulated dst are
    bit-identical to what pittile.sread / swrite produced."""
    pit = _pit()
    data, src, idx, tshape = _gather_inputs(c)
    tile = np.full(tshape, 9.0, np.float32)
    n = pit.sread(src, idx, c["group"], tile, start=c["start"])
    assert n == c["n"]
    np.testing.assert_array_equal(tile, data[c["key"] + "_tile"])
    dst = np.zeros_like(src)
    assert pit.swrite(tile, dst, idx, c["group"], start=c["start"]) == c["n"]
    np.testing.assert_array_equal(dst, data[c["key"] + "_dst"])
    acc = np.ones_like(src)
    pit.swrite(tile, acc, idx, c["group"], start=c["start"], accumulate=True)
    np.testing.assert_array_equal(acc, data[c["key"] + "_acc"])


@pytest.mark.parametrize("col_major", [False, True])
def test_gpu_sread_swrite_device_tensors_equal_reference(col_major):
    """Same known answers with CUDA tensors (source in either layout), and with a tile buffer of
    another dtype (gathered in the source dtype, cast like numpy assignment)."""
    import torch

    pit = _pit()
    for c in GATHER["cases"]:
        data, src, idx, tshape = _gather_inputs(c)
        s = torch.from_numpy(src).cuda()
        if col_major:
            s = s.t().contiguous().t()
        tile = torch.full(tshape, 9.0, dtype=torch.float32, device="cuda")
        assert pit.sread(s, idx, c["group"], tile, start=c["start"]) == c["n"]
        np.testing.assert_array_equal(tile.cpu().numpy(), data[c["key"] + "_tile"])
        tile64 = torch.full(tshape, 9.0, dtype=torch.float64, device="cuda")
        pit.sread(s, idx, c["group"], tile64, start=c["start"])
        np.testing.assert_array_equal(tile64.cpu().numpy(), data[c["key"] + "_tile"].astype(np.float64))
        acc = torch.ones_like(s)
        pit.swrite(tile, acc, idx, c["group"], start=c["start"], accumulate=True)
        np.testing.assert_array_equal(acc.cpu().numpy(), data[c["key"] + "_acc"])
        dst = torch.zeros_like(s)
        pit.swrite(tile64, dst, idx, c["group"], start=c["start"])  # f64 tile into an f32 tensor
        np.testing.assert_array_equal(dst.cpu().numpy(), data[c["key"] + "_dst"])


def test_gpu_sread_errors_match_reference():
    pit = _pit()
    c = GATHER["cases"][0]
    _, src, idx, tshape = _gather_inputs(c)
    tile = np.zeros(tshape, np.float32)
    with pytest.raises(pit.ExecError, match="out of range"):
        pit.sread(src, idx, idx.n_groups, tile)
    with pytest.raises(pit.ExecError, match="out of range"):
        pit.sread(src, idx, -1, tile)


# ------------------------------------------------------------------------------ fp32 matmul
@pytest.mark.parametrize("c", MATMUL_CASES, ids=lambda c: f"{c['i']}-{c['axis']}-{c['shape']}")
def test_gpu_fp32_matmul_equals_reference_results(c):
    """run_sparse_matmul on the GPU (fp32, FFMA path, no TF32) against the reference's recorded fp32
    result C and its f64 oracle R; ExecStats equal to the reference's recorded launches."""
    pit = _pit()
    data = np.load(GOLD / "matmul_cases.npz")
    i = c["i"]
    A, B, Cref, R = data[f"A{i}"], data[f"B{i}"], data[f"C{i}"], data[f"R{i}"]
    m, k, n = c["shape"]
    reg = pit.register_builtin_kernels()
    plan = pit.forced_plan(_bound(m, k, n), c["axis"], reg, tile_shape=tuple(c["tile"]))
    ann = pit.SparsityAnnotation((m, k), tuple(c["granularity"]), np.array(c["packed"], np.uint8))
    At = pit.DenseTensor.from_array(A, layout=plan.sparse_layout)
    stats = pit.ExecStats()
    C = pit.run_sparse_matmul(plan, At, pit.DenseTensor.from_array(B), ann if c["axis"] != "dense" else None,
                              stats=stats)
    assert isinstance(C.array, np.ndarray) and C.array.dtype == np.float32 and C.shape == (m, n)
    assert pit.max_rel_error(C, R) <= FP32_TOL
    assert pit.verify_close(C, R)
    assert pit.max_rel_error(C, Cref) <= FP32_TOL
    assert stats.launches == c["launches"]
    assert stats.gathered_micro_tiles == c["gathered"]
    # zero-completeness: where the reference has exact zeros, so do we
    np.testing.assert_array_equal(C.array[Cref == 0.0], 0.0)
    # the GPU f64 oracle is bit-identical to the reference's run_dense_reference
    np.testing.assert_array_equal(pit.run_dense_reference(At, pit.DenseTensor.from_array(B)), R)


# ----------------------------------------------------------------------- reference-written files
@pytest.mark.parametrize("c", WIRE_CASES, ids=lambda c: c["name"])
def test_gpu_replays_reference_written_files(c):
    """Load the reference's annotation text and PITT tensors, run on the GPU, compare with the
    reference's PITT result file (fp32 and f64 oracle) and its index dump, byte for byte."""
    pit = _pit()
    m, k, n = c["shape"]
    ann = pit.load_annotation(WIRE / f"{c['name']}.ann")
    A = pit.load_tensor(WIRE / f"{c['name']}_A.pitt")
    B = pit.load_tensor(WIRE / f"{c['name']}_B.pitt")
    Cref = pit.load_tensor(WIRE / f"{c['name']}_C.pitt").array
    R = pit.load_tensor(WIRE / f"{c['name']}_R.pitt").array
    reg = pit.register_builtin_kernels()
    plan = pit.forced_plan(_bound(m, k, n), c["axis"], reg, tile_shape=tuple(c["tile"]))
    stats = pit.ExecStats()
    C = pit.run_sparse_matmul(plan, A, B, ann if c["axis"] != "dense" else None, stats=stats)
    assert pit.max_rel_error(C, R) <= FP32_TOL and pit.max_rel_error(C, Cref) <= FP32_TOL
    assert stats.launches == c["launches"] and stats.gathered_micro_tiles == c["gathered"]
    if c["axis"] != "dense":
        idx = pit.build_index(ann, tuple(c["micro"]), c["axis"])
        assert pit.dump_index(idx) == (WIRE / f"{c['name']}.index").read_text()
        # value route on the device operand gives the same index (data and annotation agree)
        import torch

        Ad = torch.from_numpy(A.array).cuda() if A.layout == "row_major" else \
            torch.from_numpy(np.ascontiguousarray(A.array.T)).cuda().t()
        idx_v = pit.build_index_from_tensor(Ad, tuple(c["micro"]), c["axis"])
        assert idx_v.total <= idx.total  # a live block may hold exact zeros only by chance


def test_gpu_c1_1024_index_from_reference_annotation_file():
    """BASELINE configs[0]'s annotation (1024^2, 32x1 blocks, 90% zero, seed 1) as the reference
    wrote it: the device index equals the reference's dump, through both index routes."""
    import torch

    pit = _pit()
    ann = pit.load_annotation(WIRE / "c1_1024.ann")
    want = (WIRE / "c1_1024.index").read_text()
    assert pit.dump_index(pit.build_index(ann, (32, 1), "k")) == want
    # values masked by the annotation, detected from values on the device (bf16 column-major)
    rng = np.random.default_rng(0)
    A = rng.uniform(0.5, 1.5, (1024, 1024)).astype(np.float32) * ann.materialize()
    At = torch.from_numpy(A).to(torch.bfloat16).cuda().t().contiguous().t()
    assert pit.dump_index(pit.build_index_from_tensor(At, (32, 1), "k")) == want
