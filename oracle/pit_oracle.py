"""CPU oracle for the PIT hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this module, and only as the checker or the timed CPU baseline. The product package
(paper_2301_10936_b200) never imports it.

A numpy restatement of the reference algorithm (reference = /root/reference/pkg/src/pittile,
pure Python + numpy, no third-party algorithm beyond numpy's np.dot -> OpenBLAS sgemm for the tile
product, tiles.py:141-143). Every function cites the reference lines it follows. Pinned against
the reference itself: tests/golden/make_golden.py imports the reference in the build container
and records its outputs as fixtures; tests/test_oracle_golden.py checks this module against them.

Annotations are passed as (tensor_shape, granularity, packed) with `packed` = np.packbits of the
row-major block grid (MSB first, sparsity.py:36-48). Indexes are (counts int64[n_groups],
groups = list of int64 arrays in stored order).
"""

from __future__ import annotations

import numpy as np

PIT_DIMS = {"m": 0, "p": 0, "k": 1, "l": 1}  # index.py:25


def cdiv(a: int, b: int) -> int:
    return -(-int(a) // int(b))


# ----------------------------------------------------------------------------- annotations
def ann_bits(shape, gran, packed) -> np.ndarray:
    """sparsity.py:36-41 — unpack the block grid."""
    g0, g1 = cdiv(shape[0], gran[0]), cdiv(shape[1], gran[1])
    return np.unpackbits(np.asarray(packed, np.uint8), count=g0 * g1).astype(bool).reshape(g0, g1)


def mask_to_ann(mask, gran):
    """sparsity.py:95-106 (from_mask): block any-reduce, tails are zero padding."""
    mask = np.asarray(mask)
    s0, s1 = mask.shape
    g0, g1 = cdiv(s0, gran[0]), cdiv(s1, gran[1])
    pad = np.zeros((g0 * gran[0], g1 * gran[1]), bool)
    pad[:s0, :s1] = mask != 0
    bits = pad.reshape(g0, gran[0], g1, gran[1]).any(axis=(1, 3))
    return (s0, s1), tuple(gran), np.packbits(bits.ravel())


def random_ann(shape, gran, zero_ratio, seed):
    """sparsity.py:124-132 — one uniform draw per block, live iff draw >= zero_ratio."""
    g0, g1 = cdiv(shape[0], gran[0]), cdiv(shape[1], gran[1])
    bits = np.random.default_rng(seed).random((g0, g1)) >= zero_ratio
    return tuple(shape), tuple(gran), np.packbits(bits.ravel())


def materialize(shape, gran, packed, dtype=np.float32) -> np.ndarray:
    """sparsity.py:61-65."""
    b = ann_bits(shape, gran, packed)
    e = np.repeat(np.repeat(b, gran[0], axis=0), gran[1], axis=1)
    return e[: shape[0], : shape[1]].astype(dtype)


# ---------------------------------------------------------------------------------- index
def micro_occupancy(shape, gran, packed, micro) -> np.ndarray:
    """index.py:68-99 restated over the whole grid: micro-tile (i,j) is live iff some in-extent
    element of [i*t0, min((i+1)t0, s0)) x [j*t1, min((j+1)t1, s1)) falls in a set block.
    Evaluated at element resolution like the reference (repeat the block bits, pool per micro)."""
    t0, t1 = micro
    s0, s1 = shape
    elem = np.repeat(np.repeat(ann_bits(shape, gran, packed), gran[0], axis=0), gran[1], axis=1)[:s0, :s1]
    G0, G1 = cdiv(s0, t0), cdiv(s1, t1)
    pad = np.zeros((G0 * t0, G1 * t1), bool)
    pad[:s0, :s1] = elem
    return pad.reshape(G0, t0, G1, t1).any(axis=(1, 3))


def build_index(shape, gran, packed, micro, pit_axis):
    """index.py:102-161 with workers=1: per group (position on the non-PIT micro grid) the live
    PIT-axis coordinates in ascending order (np.nonzero order, index.py:134)."""
    micro = (int(micro[0]), int(micro[1]))
    if len(micro) != 2 or min(micro) <= 0:
        raise ValueError("micro-tile edges must be positive")
    dim = PIT_DIMS[pit_axis] if isinstance(pit_axis, str) else int(pit_axis)
    occ = micro_occupancy(shape, gran, packed, micro)
    per_group = occ.T if dim == 0 else occ  # rows = groups, columns = PIT coordinates
    groups = [np.nonzero(r)[0].astype(np.int64) for r in per_group]
    counts = np.array([g.size for g in groups], dtype=np.int64)
    return counts, groups


def build_index_from_values(values, micro, pit_axis):
    """index.py:164-173: detection on raw values with the exact test value != 0.0."""
    ann = mask_to_ann(np.asarray(values) != 0.0, (1, 1))
    return build_index(*ann, micro, pit_axis)


def dump_index(micro, pit_axis, counts, groups) -> str:
    """index.py:185-195 canonical dump."""
    lines = [f"microtile {micro[0]} {micro[1]}", f"pit_axis {pit_axis}"]
    for g, (c, coords) in enumerate(zip(counts, groups)):
        body = " ".join(str(int(x)) for x in np.sort(coords))
        lines.append(f"group {g} {int(c)}:" + (f" {body}" if body else ""))
    return "\n".join(lines) + "\n"


# -------------------------------------------------------------------------- SRead / SWrite
def sread(arr, groups, micro, pit_dim, group, tile, start=0) -> int:
    """executor.py:170-208: gather coordinates [start, start+n_slots) of a group in stored order
    into consecutive slots; zero-fill when partial or at an edge."""
    t0, t1 = micro
    d = pit_dim
    t_d, t_o = (t0, t1) if d == 0 else (t1, t0)
    n_slots = tile.shape[d] // t_d
    coords = groups[group][start : start + n_slots]
    off_o = group * t_o
    v_o = min(t_o, arr.shape[1 - d] - off_o)
    full = coords.size == n_slots and v_o == tile.shape[1 - d]
    edge = coords.size and (int(coords.max()) + 1) * t_d > arr.shape[d]
    if not full or edge:
        tile.fill(0)
    for s, c in enumerate(coords):
        e = int(c) * t_d
        v_d = min(t_d, arr.shape[d] - e)
        if d == 0:
            tile[s * t_d : s * t_d + v_d, :v_o] = arr[e : e + v_d, off_o : off_o + v_o]
        else:
            tile[:v_o, s * t_d : s * t_d + v_d] = arr[off_o : off_o + v_o, e : e + v_d]
    return int(coords.size)


def swrite(tile, arr, groups, micro, pit_dim, group, start=0, accumulate=False) -> int:
    """executor.py:211-264: mirror scatter; padded slots are never written."""
    t0, t1 = micro
    d = pit_dim
    t_d, t_o = (t0, t1) if d == 0 else (t1, t0)
    n_slots = tile.shape[d] // t_d
    coords = groups[group][start : start + n_slots]
    off_o = group * t_o
    v_o = min(t_o, arr.shape[1 - d] - off_o)
    for s, c in enumerate(coords):
        e = int(c) * t_d
        v_d = min(t_d, arr.shape[d] - e)
        if d == 0:
            piece = tile[s * t_d : s * t_d + v_d, :v_o]
            view = arr[e : e + v_d, off_o : off_o + v_o]
        else:
            piece = tile[:v_o, s * t_d : s * t_d + v_d]
            view = arr[off_o : off_o + v_o, e : e + v_d]
        if accumulate:
            view += piece
        else:
            view[...] = piece
    return int(coords.size)


# -------------------------------------------------------------------------------- matmul
def dense_reference_f64(A, B) -> np.ndarray:
    """executor.py:267-283: f64, k ascending, multiply then add (== scalar triple loop)."""
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    C = np.zeros((A.shape[0], B.shape[1]))
    tmp = np.empty_like(C)
    for k in range(A.shape[1]):
        np.multiply(A[:, k, None], B[k], out=tmp)
        C += tmp
    return C


def max_rel_error(x, y, floor=1e-6) -> float:
    """executor.py:294-300."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    if not y.size:
        return 0.0
    return float(np.max(np.abs(x - y))) / max(float(np.max(np.abs(y))), floor)


def verify_close(x, y, rtol=1e-5, atol=1e-6) -> bool:
    """executor.py:303-307."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    return True if not y.size else bool(np.max(np.abs(x - y)) <= atol + rtol * float(np.max(np.abs(y))))


def matmul_pit_k(A, B, groups, micro, tile_shape, dtype=np.float32):
    """executor.py:386-423 (single worker): for each M-block group, chunks of K_tile live k:
    gather A columns and the matching B rows, tile dot per N block, accumulate into C."""
    M_t, K_t, N_t = tile_shape
    A = np.asarray(A, dtype)
    B = np.asarray(B, dtype)
    m, n = A.shape[0], B.shape[1]
    C = np.zeros((m, n), dtype)
    t0 = micro[0]
    a_buf = np.zeros((M_t, K_t), dtype)
    for mg, ks_all in enumerate(groups):
        m0 = mg * t0
        mv = min(M_t, m - m0)
        for off in range(0, ks_all.size, K_t):
            ks = ks_all[off : off + K_t]
            a_buf.fill(0)
            a_buf[:mv, : ks.size] = A[m0 : m0 + mv][:, ks]
            b = np.zeros((K_t, n), dtype)
            b[: ks.size] = B[ks]
            for n0 in range(0, n, N_t):
                nv = min(N_t, n - n0)
                panel = np.zeros((K_t, N_t), dtype)
                panel[:, :nv] = b[:, n0 : n0 + nv]
                c = np.dot(a_buf, panel)
                C[m0 : m0 + mv, n0 : n0 + nv] += c[:mv, :nv]
    return C


def matmul_pit_m(A, B, groups, micro, tile_shape, dtype=np.float32):
    """executor.py:352-383 (single worker): for each K-block group, chunks of M_tile live rows:
    gather the rows' K-block strip, tile dot with the B K-block, scatter-accumulate into C rows.
    Each C element sums its live K-blocks in ascending order."""
    M_t, K_t, N_t = tile_shape
    A = np.asarray(A, dtype)
    B = np.asarray(B, dtype)
    m, k = A.shape
    n = B.shape[1]
    C = np.zeros((m, n), dtype)
    for kb, rows_all in enumerate(groups):
        k0 = kb * K_t
        kv = min(K_t, k - k0)
        panel = np.zeros((K_t, n), dtype)
        panel[:kv] = B[k0 : k0 + kv]
        for off in range(0, rows_all.size, M_t):
            rows = rows_all[off : off + M_t]
            a_buf = np.zeros((M_t, K_t), dtype)
            a_buf[: rows.size, :kv] = A[rows, k0 : k0 + kv]
            out = np.zeros((M_t, n), dtype)
            for n0 in range(0, n, N_t):
                nv = min(N_t, n - n0)
                p = np.zeros((K_t, N_t), dtype)
                p[:, :nv] = panel[:, n0 : n0 + nv]
                out[:, n0 : n0 + nv] = np.dot(a_buf, p)[:, :nv]
            C[rows] += out[: rows.size]
    return C


def matmul_dense(A, B, tile_shape, dtype=np.float32):
    """executor.py:426-461: dense tiling, K-blocks ascending."""
    M_t, K_t, N_t = tile_shape
    A = np.asarray(A, dtype)
    B = np.asarray(B, dtype)
    m, k = A.shape
    n = B.shape[1]
    C = np.zeros((m, n), dtype)
    for k0 in range(0, k, K_t):
        kv = min(K_t, k - k0)
        for m0 in range(0, m, M_t):
            mv = min(M_t, m - m0)
            C[m0 : m0 + mv] += np.dot(A[m0 : m0 + mv, k0 : k0 + kv], B[k0 : k0 + kv])
    return C


def run_sparse_matmul(A, B, ann, pit_axis, tile_shape, dtype=np.float32):
    """executor.py:519-537: build the index from the annotation at the plan's micro-tile
    (policy.py:69-105: tile projection with extent 1 along the PIT axis), then execute."""
    M_t, K_t, _ = tile_shape
    if pit_axis == "dense":
        return matmul_dense(A, B, tile_shape, dtype)
    micro = (1, K_t) if pit_axis == "m" else (M_t, 1)
    _, groups = build_index(*ann, micro, pit_axis)
    if pit_axis == "m":
        return matmul_pit_m(A, B, groups, micro, tile_shape, dtype)
    return matmul_pit_k(A, B, groups, micro, tile_shape, dtype)


def plan_launches(counts, pit_axis, tile_shape, n) -> int:
    """policy.py:160-184 for sparse matmul plans."""
    M_t, K_t, N_t = tile_shape
    chunk = M_t if pit_axis == "m" else K_t
    return int(np.sum(-(-np.asarray(counts) // chunk))) * cdiv(n, N_t)


# ------------------------------------------------------------------------------------- MoE
def switch_route(logits):
    """Top-1 routing: expert = argmax (first maximum, like np.argmax), gate = softmax prob of it.
    The expert -> token index is build_index(from_mask(onehot, (1,1)), (1,1), "m") (index.py:102-173,
    sparsity.py:95-106): groups = experts, coordinates = tokens ascending."""
    lg = np.asarray(logits, np.float64)
    expert = np.argmax(lg, axis=1)
    mx = lg[np.arange(lg.shape[0]), expert]
    gate = 1.0 / np.exp(lg - mx[:, None]).sum(axis=1)
    onehot = np.zeros_like(lg, dtype=bool)
    onehot[np.arange(lg.shape[0]), expert] = True
    counts, groups = build_index(*mask_to_ann(onehot, (1, 1)), (1, 1), "m")
    return expert, gate, counts, groups


def switch_forward(x, logits, w1, w2, round_hidden=None):
    """Switch FFN: out[t] = gate[t] * relu(x[t] @ W1[e]) @ W2[e] in f64, per expert over its token
    group (SRead rows -> two dense products -> SWrite * gate). `round_hidden` optionally rounds the
    hidden activations (e.g. to bf16) to mirror a low-precision intermediate."""
    x = np.asarray(x, np.float64)
    expert, gate, counts, groups = switch_route(logits)
    out = np.zeros((x.shape[0], np.asarray(w2).shape[2]))
    for e, toks in enumerate(groups):
        if toks.size == 0:
            continue
        h = np.maximum(x[toks] @ np.asarray(w1[e], np.float64), 0.0)
        if round_hidden is not None:
            h = round_hidden(h)
        out[toks] = gate[toks, None] * (h @ np.asarray(w2[e], np.float64))
    return out


# ------------------------------------------------------------------------------ reduce_sum
def reduce_sum(A, ann, pit_axis, tile_shape, dtype=np.float32):
    """executor.py:540-613 (single worker): pit:l gathers each row's live elements (micro (1,1),
    policy.py:95-97), pit:p gathers live rows per L-block (micro (1, L)); dense sums tiles.
    Tile sums are accumulated into C in the reference's chunk order."""
    P, L = tile_shape
    A = np.asarray(A, dtype)
    p, l = A.shape
    C = np.zeros(p, dtype)
    if pit_axis == "dense":
        for p0 in range(0, p, P):
            for l0 in range(0, l, L):
                C[p0 : p0 + P] += A[p0 : p0 + P, l0 : l0 + L].sum(axis=1)
        return C
    if pit_axis == "p":
        _, groups = build_index(*ann, (1, L), "p")
        for g, rows in enumerate(groups):
            for off in range(0, rows.size, P):
                r = rows[off : off + P]
                C[r] += A[r, g * L : (g + 1) * L].sum(axis=1)
        return C
    _, groups = build_index(*ann, (1, 1), "l")
    for p0 in range(0, p, P):
        rows = range(p0, min(p0 + P, p))
        chunks = max((-(-groups[r].size // L) for r in rows), default=0)
        for c in range(chunks):
            for r in rows:
                seg = groups[r][c * L : (c + 1) * L]
                if seg.size:
                    C[r] += A[r, seg].sum()
    return C


# ------------------------------------------------------------- output-sparse matmul (8(f)3)
def sddmm(A, B, ann, out, gate=None):
    """Output-sparse product: out[i, j] = (A . B)[i, j] (f64, k ascending like run_dense_reference,
    executor.py:267-283) for every element whose annotation block of C is live (sparsity.py:61-65
    materialize); elements of dead blocks keep their value. With `gate`, stored elements are 0 where
    gate <= 0. The reference documents this plan (README.md:150-153) without executing
    it; this is its definition, not a port."""
    live = materialize(*ann, dtype=np.float64).astype(bool)
    prod = dense_reference_f64(A, B)
    if gate is not None:
        prod = np.where(np.asarray(gate, np.float64) > 0, prod, 0.0)
    res = np.array(out, dtype=np.float64, copy=True)
    res[live] = prod[live]
    return res, live
