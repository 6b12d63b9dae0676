"""Generate golden fixtures by running the REFERENCE implementation (pittile) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed here as small fixtures:
  index_cases.json   annotation (packed bits) -> canonical dump_index text, counts, cover_count
  value_cases.npz    raw values (incl. -0.0 / NaN / denormals) -> dump text (build_index_from_tensor)
  gather_cases.npz   sread / swrite known answers
  matmul_cases.npz   run_sparse_matmul fp32 results + the f64 oracle for pit:m / pit:k / dense
  plan_cases.json    get_micro_tile, plan_launches, cover table (PAPER.md:1072-1094 configs)
  wire/              files WRITTEN BY THE REFERENCE in its own formats: annotation text
                     (sparsity.py:135-144), PITT tensors (executor.py:93-102), index dumps
                     (index.py:185-195) and a `pittile bench` CSV (cli.py:330) - read back by the
                     package and replayed on the GPU (tests/test_wire_formats.py, test_gpu_golden.py)
Everything is seeded; rerunning reproduces the files byte for byte.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

import pittile as pt  # noqa: E402

OUT = Path(__file__).resolve().parent
MATMUL = "C[m,n] += A[m,k] * B[k,n]"


def bound(m, k, n):
    return pt.bind_extents(pt.parse_expr(MATMUL), dict(m=m, k=k, n=n))


def index_cases():
    rng = np.random.default_rng(20240)
    cases = []
    fixed = [
        ((64, 64), (1, 1), (1, 8), "m", 0.7),
        ((45, 70), (3, 2), (1, 32), "m", 0.6),
        ((45, 70), (3, 2), (16, 1), "k", 0.6),
        ((1024, 1024), (32, 1), (32, 1), "k", 0.9),
        ((1024, 1024), (1, 32), (1, 32), "m", 0.9),
        ((1, 1), (1, 1), (1, 1), "m", 0.4),
        ((200, 1), (1, 1), (16, 1), "k", 0.4),
        ((1, 200), (1, 1), (1, 32), "m", 0.4),
        ((512, 768), (1, 768), (1, 64), "m", 0.45),
        ((256, 256), (32, 64), (1, 64), "m", 0.9),
        ((256, 256), (32, 64), (32, 1), "k", 0.9),
    ]
    for t in range(60):
        shape = (int(rng.integers(1, 200)), int(rng.integers(1, 200)))
        gran = (int(rng.integers(1, 6)), int(rng.integers(1, 6)))
        micro = (int(rng.integers(1, 24)), int(rng.integers(1, 24)))
        axis = ["m", "k"][int(rng.integers(2))]
        ratio = float(rng.choice([0.0, 0.3, 0.7, 0.95, 1.0]))
        fixed.append((shape, gran, micro, axis, ratio))
    for i, (shape, gran, micro, axis, ratio) in enumerate(fixed):
        seed = 1 if shape == (1024, 1024) else 1000 + i
        ann = pt.random_annotation(shape, gran, ratio, seed=seed)
        idx = pt.build_index(ann, micro, axis)
        cases.append(
            dict(
                shape=list(shape),
                granularity=list(gran),
                micro=list(micro),
                axis=axis,
                zero_ratio=ratio,
                seed=seed,
                packed=ann.packed.tolist(),
                counts=idx.counts.tolist(),
                total=idx.total,
                cover=pt.cover_count(ann, micro, axis),
                dump=pt.dump_index(idx),
            )
        )
    (OUT / "index_cases.json").write_text(json.dumps(cases, separators=(",", ":")))


def value_cases():
    rng = np.random.default_rng(77)
    arrays, dumps = {}, []
    specs = [((40, 30), (4, 5), "m"), ((40, 30), (4, 5), "k"), ((64, 96), (1, 32), "m"), ((96, 64), (32, 1), "k"),
             ((33, 17), (1, 1), "m"), ((8, 64), (1, 32), "m")]
    for i, (shape, micro, axis) in enumerate(specs):
        v = rng.standard_normal(shape).astype(np.float32)
        v[rng.random(shape) > 0.05] = 0.0
        if i == 5:
            v[:] = 0.0
            v[1, 3] = -0.0
            v[2, 40] = np.float32(1e-45)
            v[4, 10] = np.nan
            v[6, 63] = -np.inf
        arrays[f"v{i}"] = v
        idx = pt.build_index_from_tensor(v, micro, axis)
        dumps.append(dict(key=f"v{i}", micro=list(micro), axis=axis, dump=pt.dump_index(idx)))
    np.savez_compressed(OUT / "value_cases.npz", **arrays)
    (OUT / "value_cases.json").write_text(json.dumps(dumps))


def gather_cases():
    rng = np.random.default_rng(99)
    out = {}
    meta = []
    specs = [((16, 8), (1, 8), "m", (4, 8)), ((16, 10), (1, 4), "m", (3, 4)), ((6, 10), (6, 1), "k", (6, 4)),
             ((13, 11), (3, 2), "m", (7, 2)), ((13, 11), (3, 2), "k", (3, 5)), ((9, 9), (2, 2), "m", (4, 2))]
    for i, (shape, micro, axis, tshape) in enumerate(specs):
        src = rng.standard_normal(shape).astype(np.float32)
        src[rng.random(shape) > 0.5] = 0.0
        idx = pt.build_index(pt.from_mask(src, (1, 1)), micro, axis)
        for g in range(idx.n_groups):
            for start in (0, 1):
                tile = np.full(tshape, 9.0, np.float32)
                n = pt.sread(src, idx, g, tile, start=start)
                dst = np.zeros_like(src)
                pt.swrite(tile, dst, idx, g, start=start)
                acc = np.ones_like(src)
                pt.swrite(tile, acc, idx, g, start=start, accumulate=True)
                key = f"c{i}_g{g}_s{start}"
                out[key + "_tile"] = tile
                out[key + "_dst"] = dst
                out[key + "_acc"] = acc
                meta.append(dict(key=key, case=i, group=g, start=start, n=n))
        out[f"src{i}"] = src
    np.savez_compressed(OUT / "gather_cases.npz", **out)
    (OUT / "gather_cases.json").write_text(
        json.dumps(dict(specs=[[list(s), list(m), a, list(t)] for s, m, a, t in specs], cases=meta))
    )


def matmul_cases():
    rng = np.random.default_rng(31)
    reg = pt.register_builtin_kernels()
    out, meta = {}, []
    specs = [
        ((64, 64, 64), "m", (16, 32, 128), (1, 64), 0.5),
        ((45, 70, 51), "m", (16, 32, 128), (3, 2), 0.6),
        ((45, 70, 51), "k", (16, 32, 128), (3, 2), 0.6),
        ((45, 70, 51), "dense", (32, 64, 32), (3, 2), 0.6),
        ((96, 128, 64), "k", (32, 64, 32), (32, 1), 0.9),
        ((128, 96, 160), "m", (8, 32, 128), (1, 96), 0.5),
        ((1, 200, 1), "k", (16, 32, 128), (1, 1), 0.4),
        ((200, 1, 1), "m", (16, 32, 128), (1, 1), 0.4),
        ((1, 1, 200), "dense", (16, 32, 128), (1, 1), 0.4),
        ((128, 128, 96), "k", (32, 32, 32), (8, 1), 0.95),
        ((96, 96, 96), "m", (32, 64, 32), (1, 1), 0.0),
    ]
    for i, ((m, k, n), axis, tile, gran, ratio) in enumerate(specs):
        ann = pt.random_annotation((m, k), gran, ratio, seed=500 + i)
        A = rng.standard_normal((m, k)).astype(np.float32) * ann.materialize()
        B = rng.standard_normal((k, n)).astype(np.float32)
        plan = pt.forced_plan(bound(m, k, n), axis, reg, tile_shape=tile)
        At = pt.DenseTensor.from_array(A, layout=plan.sparse_layout)
        stats = pt.ExecStats()
        C = pt.run_sparse_matmul(plan, At, pt.DenseTensor.from_array(B), ann if axis != "dense" else None, stats=stats)
        out[f"A{i}"] = A
        out[f"B{i}"] = B
        out[f"C{i}"] = C.array
        out[f"R{i}"] = pt.run_dense_reference(At, pt.DenseTensor.from_array(B))
        meta.append(dict(i=i, shape=[m, k, n], axis=axis, tile=list(tile), granularity=list(gran), zero_ratio=ratio,
                         seed=500 + i, packed=ann.packed.tolist(), launches=stats.launches,
                         gathered=stats.gathered_micro_tiles))
    np.savez_compressed(OUT / "matmul_cases.npz", **out)
    (OUT / "matmul_cases.json").write_text(json.dumps(meta))


def plan_cases():
    reg = pt.register_builtin_kernels()
    micro = {f"{'x'.join(map(str, t))}:{a}": list(pt.get_micro_tile("matmul", t, a)) for t in
             ((16, 32, 128), (8, 32, 128), (32, 64, 32), (32, 32, 32)) for a in ("m", "k")}
    table = []
    for gran, ratio, mt in [((2, 1), 0.95, (16, 1)), ((2, 1), 0.99, (8, 1)), ((4, 1), 0.95, (16, 1)),
                            ((4, 1), 0.99, (16, 1)), ((8, 1), 0.95, (8, 1)), ((8, 1), 0.99, (32, 1)),
                            ((32, 1), 0.95, (32, 1)), ((32, 1), 0.99, (32, 1))]:
        ann = pt.random_annotation((4096, 4096), gran, ratio, seed=20_000 + gran[0])
        table.append(dict(granularity=list(gran), zero_ratio=ratio, micro=list(mt),
                          cover=pt.cover_count(ann, mt, "m"), seed=20_000 + gran[0]))
    launches = []
    for trial in range(10):
        r = np.random.default_rng(trial)
        m, k, n = (int(x) for x in r.integers(10, 200, size=3))
        ann = pt.random_annotation((m, k), (2, 3), 0.7, seed=trial)
        for axis, tile in (("m", (16, 32, 128)), ("k", (32, 64, 32)), ("dense", (8, 32, 128))):
            plan = pt.forced_plan(bound(m, k, n), axis, reg, tile_shape=tile)
            launches.append(dict(shape=[m, k, n], seed=trial, axis=axis, tile=list(tile),
                                 launches=pt.plan_launches(plan, ann if axis != "dense" else None)))
    (OUT / "plan_cases.json").write_text(json.dumps(dict(micro=micro, cover_table=table, launches=launches)))


def reduce_cases():
    rng = np.random.default_rng(61)
    reg = pt.register_builtin_kernels()
    out, meta = {}, []
    for i, (p_, l_, axis) in enumerate([(70, 200, "l"), (70, 200, "p"), (70, 200, "dense"), (8, 16, "l"),
                                         (33, 129, "p"), (1, 300, "l")]):
        expr = pt.bind_extents(pt.parse_expr("C[p] += A[p,l]"), dict(p=p_, l=l_))
        lengths = [int(x) for x in rng.integers(0, l_ + 1, p_)]
        ann = pt.from_ragged_lengths(lengths, [p_, l_])
        A = rng.standard_normal((p_, l_)).astype(np.float32) * ann.materialize()
        plan = pt.forced_plan(expr, axis, reg)
        stats = pt.ExecStats()
        C = pt.run_sparse_reduce_sum(plan, pt.DenseTensor.from_array(A), ann if axis != "dense" else None, stats=stats)
        out[f"A{i}"] = A
        out[f"C{i}"] = C.array
        meta.append(dict(i=i, shape=[p_, l_], axis=axis, lengths=lengths, packed=ann.packed.tolist(),
                         launches=stats.launches, gathered=stats.gathered_micro_tiles))
    np.savez_compressed(OUT / "reduce_cases.npz", **out)
    (OUT / "reduce_cases.json").write_text(json.dumps(meta))


def wire_cases():
    """Reference-written files in the reference's own formats."""
    wire = OUT / "wire"
    wire.mkdir(exist_ok=True)
    rng = np.random.default_rng(4242)
    reg = pt.register_builtin_kernels()
    specs = [  # name, (m, k, n), axis, tile, granularity, zero ratio
        ("c1_pitk", (256, 256, 128), "k", (32, 64, 32), (32, 1), 0.9),
        ("pitm_1x32", (128, 256, 96), "m", (16, 32, 128), (1, 32), 0.9),
        ("blocks_32x64", (256, 256, 64), "m", (32, 64, 32), (32, 64), 0.8),
        ("ragged_pitk", (45, 70, 51), "k", (16, 32, 128), (3, 2), 0.6),
        ("dense", (64, 96, 80), "dense", (32, 64, 32), (1, 1), 0.0),
    ]
    meta = []
    for i, (name, (m, k, n), axis, tile, gran, ratio) in enumerate(specs):
        ann = pt.random_annotation((m, k), gran, ratio, seed=900 + i)
        pt.save_annotation(ann, wire / f"{name}.ann")
        A = rng.standard_normal((m, k)).astype(np.float32) * ann.materialize()
        B = rng.standard_normal((k, n)).astype(np.float32)
        plan = pt.forced_plan(bound(m, k, n), axis, reg, tile_shape=tile)
        At = pt.DenseTensor.from_array(A, layout=plan.sparse_layout)
        stats = pt.ExecStats()
        C = pt.run_sparse_matmul(plan, At, pt.DenseTensor.from_array(B), ann if axis != "dense" else None,
                                 stats=stats)
        pt.save_tensor(At, wire / f"{name}_A.pitt")
        pt.save_tensor(pt.DenseTensor.from_array(B), wire / f"{name}_B.pitt")
        pt.save_tensor(C, wire / f"{name}_C.pitt")
        pt.save_tensor(pt.DenseTensor(pt.run_dense_reference(At, pt.DenseTensor.from_array(B))),
                       wire / f"{name}_R.pitt")
        if axis != "dense":
            idx = pt.build_index(ann, plan.micro_tile, axis)
            (wire / f"{name}.index").write_text(pt.dump_index(idx))
        meta.append(dict(name=name, shape=[m, k, n], axis=axis, tile=list(tile), micro=list(plan.micro_tile or ()),
                         granularity=list(gran), zero_ratio=ratio, seed=900 + i,
                         launches=stats.launches, gathered=stats.gathered_micro_tiles))
    # the C1 annotation itself (BASELINE configs[0]: 1024^2, 32x1 blocks, 90% zero, seed 1)
    c1 = pt.random_annotation((1024, 1024), (32, 1), 0.9, seed=1)
    pt.save_annotation(c1, wire / "c1_1024.ann")
    (wire / "c1_1024.index").write_text(pt.dump_index(pt.build_index(c1, (32, 1), "k")))
    (wire / "wire_cases.json").write_text(json.dumps(meta, indent=1))


def wire_cli():
    """The reference CLI's own outputs: a CPU cost table (`pittile profile`, tiles.py:224-253) and a
    sparsity-sweep CSV (`pittile bench`, cli.py:271-345). Timings differ per run; the files pin the
    formats, not the numbers."""
    import os
    import subprocess

    wire = OUT / "wire"
    env = dict(os.environ, PYTHONPATH=str(REF))
    prof = wire / "pittile_cpu.prof"
    subprocess.run([sys.executable, "-m", "pittile", "profile", "--reps", "3", "-o", str(prof)], check=True, env=env)
    subprocess.run([sys.executable, "-m", "pittile", "bench", "--expr", MATMUL, "--shape", "m=256,k=256,n=256",
                    "--random", "32x1:0.9", "--ratios", "0.5,0.9", "--profile", str(prof), "--csv",
                    str(wire / "pittile_bench.csv")], check=True, env=env)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate only the named fixture sets, e.g. `make_golden.py wire_cases`
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    wire_cases()
    reduce_cases()
    index_cases()
    value_cases()
    gather_cases()
    matmul_cases()
    plan_cases()
    print("golden fixtures written to", OUT)
