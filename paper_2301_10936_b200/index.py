"""Online sparsity detection: micro-tile indexes built on the GPU.

Mirrors ``pittile.index`` (reference pkg/src/pittile/index.py:32-195). ``build_index`` and
``build_index_from_tensor`` run the K1 detection kernels (csrc/pit_detect.cu) through the C ABI:
an HBM-bound occupancy scan followed by an ordered per-group compaction. Groups come back in
ascending order, i.e. exactly the reference's ``workers=1`` order — stronger than the
reference's "unordered" contract (index.py:1-11), so ``canonicalize`` is the identity on them.

The index lives on the device (int32 counts / slots plus the group-major occupancy bitmap).
``counts`` / ``slots`` materialise int64 host copies on first access; those copies are read-only
while the device copy is authoritative. ``canonicalize`` returns a host-authoritative, writable
index (the reference tests reorder slots in place, test_executor.py:233-265), which is uploaded
again when it is next executed.
"""

from __future__ import annotations

from typing import Optional, Union

import numpy as np

from . import _device, _lib
from .sparsity import SparsityAnnotation

PIT_DIMS = {"m": 0, "p": 0, "k": 1, "l": 1}


class IndexBuildError(ValueError):
    pass


def _pit_dim(pit_axis: Union[str, int]) -> int:
    if isinstance(pit_axis, (int, np.integer)) and not isinstance(pit_axis, bool):
        if int(pit_axis) not in (0, 1):
            raise IndexBuildError(f"pit dimension must be 0 or 1, got {pit_axis}")
        return int(pit_axis)
    if pit_axis not in PIT_DIMS:
        raise IndexBuildError(f"unknown permuted axis {pit_axis!r}")
    return PIT_DIMS[pit_axis]


def _micro(micro_tile) -> tuple[int, int]:
    mt = tuple(int(t) for t in micro_tile)
    if len(mt) != 2:
        raise IndexBuildError(f"micro-tile rank {len(mt)} does not match annotation rank 2")
    if min(mt) <= 0:
        raise IndexBuildError(f"micro-tile edges must be positive, got {mt}")
    return mt  # type: ignore[return-value]


def _geometry(shape, micro, dim) -> tuple[int, int, int]:
    g0 = -(-int(shape[0]) // micro[0])
    g1 = -(-int(shape[1]) // micro[1])
    pit_grid, n_groups = (g0, g1) if dim == 0 else (g1, g0)
    return n_groups, pit_grid, -(-pit_grid // 32)


class MicroTileIndex:
    """Per group (position along the non-PIT micro grid), the live PIT-axis micro coordinates."""

    def __init__(self, micro_tile, pit_axis, pit_dim, pit_grid, n_groups, *, shape=None, buf=None, counts=None,
                 slots=None):
        self.micro_tile = tuple(micro_tile)
        self.pit_axis = pit_axis
        self.pit_dim = pit_dim
        self.pit_grid = int(pit_grid)
        self._n_groups = int(n_groups)
        self.shape = shape  # operand shape the index was built for (None if unknown)
        # device storage: one int32 buffer = counts [n_groups] | slots [n_groups*pit_grid] | occ [n_groups*WG]
        self._buf = buf
        self._occ_valid = buf is not None
        self._union = None
        self._counts = counts
        self._slots = slots
        self._host_authoritative = counts is not None

    @property
    def words_per_group(self) -> int:
        return -(-self.pit_grid // 32)

    def _ptrs(self):
        base = self._buf.data_ptr()
        ng, pg = self._n_groups, self.pit_grid
        return base, base + 4 * ng, base + 4 * (ng + ng * pg)

    @property
    def _counts_dev(self):
        return self._buf[: self._n_groups]

    @property
    def _slots_dev(self):
        ng, pg = self._n_groups, self.pit_grid
        return self._buf[ng : ng + ng * pg].view(ng, pg)

    @property
    def _occ_dev(self):
        ng, pg = self._n_groups, self.pit_grid
        return self._buf[ng + ng * pg :].view(ng, self.words_per_group)

    # ------------------------------------------------------------------ host view
    @property
    def n_groups(self) -> int:
        return self._n_groups

    def _materialize(self) -> None:
        if self._counts is None:
            counts = _device.to_host(self._counts_dev).astype(np.int64)
            slots = _device.to_host(self._slots_dev).astype(np.int64).reshape(self._n_groups, self.pit_grid)
            for g, c in enumerate(counts):  # entries past counts[g] are unspecified: zero them for a clean view
                slots[g, c:] = 0
            counts.setflags(write=False)
            slots.setflags(write=False)
            self._counts, self._slots = counts, slots

    @property
    def counts(self) -> np.ndarray:
        self._materialize()
        return self._counts

    @property
    def slots(self) -> np.ndarray:
        self._materialize()
        return self._slots

    @property
    def total(self) -> int:
        return int(self.counts.sum())

    def group(self, g: int) -> np.ndarray:
        return self.slots[g, : self.counts[g]]

    # ---------------------------------------------------------------- device view
    def device_arrays(self):
        """(counts int32 [n_groups], slots int32 [n_groups, pit_grid]) on the current device."""
        import torch

        if self._host_authoritative:
            dev = _device.require_cuda()
            self._check_host_entries()
            counts = torch.from_numpy(np.ascontiguousarray(self._counts, dtype=np.int32)).to(dev)
            slots = torch.from_numpy(np.ascontiguousarray(self._slots, dtype=np.int32)).to(dev)
            return counts, slots
        return self._counts_dev, self._slots_dev

    def _check_host_entries(self) -> None:
        """A host-authoritative index may have been edited by the caller (the reference's tests
        write slots directly). The gathered-K kernels trust every coordinate they are given, so
        reject what the reference's executor rejects before anything is uploaded
        (executor.py:200-204: "micro-tile coordinate out of range")."""
        from .executor import ExecError

        counts = np.asarray(self._counts)
        slots = np.asarray(self._slots).reshape(self._n_groups, self.pit_grid)
        if counts.size and (int(counts.min()) < 0 or int(counts.max()) > self.pit_grid):
            raise ExecError("micro-tile coordinate out of range: group count outside [0, pit_grid]")
        live = np.arange(self.pit_grid)[None, :] < counts[:, None]
        vals = slots[live]
        if vals.size and (int(vals.min()) < 0 or int(vals.max()) >= self.pit_grid):
            raise ExecError("micro-tile coordinate out of range")

    def device_ptrs(self):
        """(counts, slots) device pointers plus the tensors keeping them alive."""
        if self._host_authoritative:
            c, sl = self.device_arrays()
            return c.data_ptr(), sl.data_ptr(), (c, sl)
        pc, ps, _ = self._ptrs()
        return pc, ps, (self._buf,)

    def occupancy_words(self):
        """Group-major occupancy bitmap (int32 storage of uint32 words) on the device."""
        import torch

        if self._occ_valid and not self._host_authoritative:
            return self._occ_dev
        dev = _device.require_cuda()
        counts, slots = self.device_arrays()
        wg = -(-self.pit_grid // 32)
        occ = torch.empty((self._n_groups, wg), dtype=torch.int32, device=dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        lib = _lib.load()
        _device.check(lib.pit_index_occupancy(counts.data_ptr(), slots.data_ptr(), self._n_groups, self.pit_grid,
                                              occ.data_ptr(), bad.data_ptr(), _device.stream_ptr()))
        if int(bad.item()):
            from .executor import ExecError

            raise ExecError("micro-tile coordinate out of range")
        return occ

    def union_coords(self):
        """(coords int32 [pit_grid], n int32 [1]) on the device: every coordinate live in any group."""
        import torch

        if self._union is not None and not self._host_authoritative:
            return self._union
        if self._n_groups == 1 and not self._host_authoritative:
            # one group (row-uniform micro-tiles spanning K, e.g. BERT's (1, 768)): the union is that
            # group's ascending coordinates — no union / compaction launches
            self._union = (self._slots_dev[0], self._counts_dev[:1])
            return self._union
        dev = _device.require_cuda()
        occ = self.occupancy_words()
        wg = -(-self.pit_grid // 32)
        ws = torch.empty(max(wg, 1), dtype=torch.int32, device=dev)
        rows = torch.empty(max(self.pit_grid, 1), dtype=torch.int32, device=dev)
        n = torch.zeros(1, dtype=torch.int32, device=dev)
        lib = _lib.load()
        _device.check(lib.pit_index_union(occ.data_ptr(), self._n_groups, self.pit_grid, ws.data_ptr(),
                                          rows.data_ptr(), n.data_ptr(), _device.stream_ptr()))
        res = (rows, n)
        if not self._host_authoritative:
            self._union = res
        return res

    def transposed(self) -> "MicroTileIndex":
        """The same index for the transposed operand: micro-tile (t0,t1) -> (t1,t0), pit axis m <-> k,
        identical groups and coordinates (no copy, shares the device buffer). E.g. the (1,32) pit:m
        index of activations H is the (32,1) pit:k index of H^T used by the weight-gradient
        product H^T.dY — one detection serves forward and backward."""
        axis = {"m": "k", "k": "m", "p": "l", "l": "p"}.get(self.pit_axis, self.pit_axis)
        shape = None if self.shape is None else (self.shape[1], self.shape[0])
        t = MicroTileIndex((self.micro_tile[1], self.micro_tile[0]), axis, 1 - self.pit_dim, self.pit_grid,
                           self._n_groups, shape=shape, buf=self._buf, counts=self._counts, slots=self._slots)
        t._occ_valid = self._occ_valid
        t._host_authoritative = self._host_authoritative
        return t

    def __repr__(self) -> str:
        return (f"MicroTileIndex(micro_tile={self.micro_tile}, pit_axis={self.pit_axis!r}, "
                f"n_groups={self._n_groups}, pit_grid={self.pit_grid})")


def _empty_index(micro, axis, dim, shape):
    import torch

    dev = _device.require_cuda()
    n_groups, pit_grid, wg = _geometry(shape, micro, dim)
    buf = torch.empty(n_groups * (1 + pit_grid + wg), dtype=torch.int32, device=dev)
    return MicroTileIndex(micro, axis, dim, pit_grid, n_groups, shape=tuple(shape), buf=buf)


def _axis_name(pit_axis, dim) -> str:
    return pit_axis if isinstance(pit_axis, str) else ("m" if dim == 0 else "k")


def build_index(ann: SparsityAnnotation, micro_tile, pit_axis: Union[str, int], workers: int = 1) -> MicroTileIndex:
    """Detect live micro-tiles of an annotation and index them per group (index.py:102-161).

    ``workers`` is accepted for API compatibility; the scan is one GPU launch.
    """
    import torch

    micro = _micro(micro_tile)
    if workers < 1:
        raise IndexBuildError("workers must be >= 1")
    dim = _pit_dim(pit_axis)
    idx = _empty_index(micro, _axis_name(pit_axis, dim), dim, ann.tensor_shape)
    if isinstance(ann.packed, torch.Tensor):  # SparsityAnnotation.on_device(): no copy, capturable
        packed = ann.packed
        if packed.dtype != torch.uint8 or not packed.is_cuda:
            raise IndexBuildError("device annotation bits must be a CUDA uint8 tensor")
    else:
        packed = torch.from_numpy(np.ascontiguousarray(ann.packed, dtype=np.uint8)).to(idx._buf.device)
    lib = _lib.load()
    s0, s1 = ann.tensor_shape
    g0, g1 = ann.granularity
    pc, ps, po = idx._ptrs()
    _device.check(lib.pit_build_index(packed.data_ptr(), s0, s1, g0, g1, micro[0], micro[1], dim, po, pc, ps,
                                      _device.stream_ptr()), IndexBuildError)
    return idx


def build_occupancy(ann: SparsityAnnotation, micro_tile, pit_axis: Union[str, int]):
    """Only the group-major occupancy bitmap of ``build_index`` (int32 storage [n_groups, words]):
    one detection launch, no compaction — for consumers that test liveness, not list coordinates
    (the output-sparse epilogue)."""
    import torch

    micro = _micro(micro_tile)
    dim = _pit_dim(pit_axis)
    n_groups, pit_grid, wg = _geometry(ann.tensor_shape, micro, dim)
    dev = _device.require_cuda()
    occ = torch.empty((n_groups, max(wg, 1)), dtype=torch.int32, device=dev)
    if isinstance(ann.packed, torch.Tensor):
        packed = ann.packed
    else:
        packed = torch.from_numpy(np.ascontiguousarray(ann.packed, dtype=np.uint8)).to(dev)
    s0, s1 = ann.tensor_shape
    g0, g1 = ann.granularity
    _device.check(_lib.load().pit_build_index(packed.data_ptr(), s0, s1, g0, g1, micro[0], micro[1], dim,
                                              occ.data_ptr(), None, None, _device.stream_ptr()), IndexBuildError)
    return occ


def build_index_from_tensor(values, micro_tile, pit_axis: Union[str, int], workers: int = 1) -> MicroTileIndex:
    """Detection directly on raw values with the exact test ``value != 0.0`` (index.py:164-173).

    ``values`` may be a host array (uploaded) or a CUDA tensor (scanned in place, row- or
    column-major).
    """
    import torch

    micro = _micro(micro_tile)
    if workers < 1:
        raise IndexBuildError("workers must be >= 1")
    dim = _pit_dim(pit_axis)
    if not isinstance(values, torch.Tensor):
        values = np.asarray(values)
    if values.ndim != 2:
        raise IndexBuildError("tensor detection supports rank-2 values")
    x = _device.to_device(values)
    if x.dtype not in (torch.float32, torch.float64, torch.bfloat16, torch.float16, torch.uint8, torch.bool):
        x = (x != 0).to(torch.uint8)
    s0, s1 = int(x.shape[0]), int(x.shape[1])
    st0, st1 = x.stride()
    if not (st1 == 1 or st0 == 1):
        x = x.contiguous()
        st0, st1 = x.stride()
    idx = _empty_index(micro, _axis_name(pit_axis, dim), dim, (s0, s1))
    lib = _lib.load()
    pc, ps, po = idx._ptrs()
    _device.check(lib.pit_build_index_from_tensor(x.data_ptr(), _device.dtype_code(x), s0, s1, st0, st1, micro[0],
                                                  micro[1], dim, po, pc, ps, _device.stream_ptr()), IndexBuildError)
    return idx


def index_from_arrays(micro_tile, pit_axis, counts, slots, pit_grid: Optional[int] = None) -> MicroTileIndex:
    """Host-authoritative index from explicit counts / slots (e.g. a reordered copy)."""
    counts = np.array(counts, dtype=np.int64)
    slots = np.array(slots, dtype=np.int64)
    dim = _pit_dim(pit_axis)
    pg = int(pit_grid) if pit_grid is not None else slots.shape[1]
    return MicroTileIndex(tuple(micro_tile), _axis_name(pit_axis, dim), dim, pg, counts.shape[0],
                          counts=counts, slots=slots.reshape(counts.shape[0], pg))


def canonicalize(idx: MicroTileIndex) -> MicroTileIndex:
    """Ascending coordinates per group; returns a writable, host-authoritative copy."""
    counts = np.array(idx.counts, dtype=np.int64)
    slots = np.array(idx.slots, dtype=np.int64)
    for g in range(idx.n_groups):
        c = counts[g]
        slots[g, :c] = np.sort(slots[g, :c])
    out = MicroTileIndex(idx.micro_tile, idx.pit_axis, idx.pit_dim, idx.pit_grid, idx.n_groups, shape=idx.shape,
                         counts=counts, slots=slots)
    return out


def dump_index(idx: MicroTileIndex) -> str:
    """Canonical text form (index.py:185-195): independent of storage order."""
    out = [f"microtile {idx.micro_tile[0]} {idx.micro_tile[1]}", f"pit_axis {idx.pit_axis}"]
    for g in range(idx.n_groups):
        coords = " ".join(str(int(c)) for c in np.sort(idx.group(g)))
        out.append(f"group {g} {int(idx.counts[g])}:" + (f" {coords}" if coords else ""))
    return "\n".join(out) + "\n"


def cover_counts_device(ann: SparsityAnnotation, candidates) -> list:
    """Per-group live micro-tile counts for many (micro_tile, pit_dim) candidates in one device pass
    over the annotation (pit_cover_counts): what plan selection needs from detection, without
    building any index. Returns one int64 numpy array per candidate."""
    import torch

    dev = _device.require_cuda()
    cands = [(_micro(m), int(d)) for m, d in candidates]
    geo = [_geometry(ann.tensor_shape, m, d) for m, d in cands]
    total = sum(ng for ng, _, _ in geo)
    ws = max([ng * wg for ng, _, wg in geo] + [1])
    packed = torch.from_numpy(np.ascontiguousarray(ann.packed, dtype=np.uint8)).to(dev)
    occ = torch.empty(ws, dtype=torch.int32, device=dev)
    out = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    flat = np.array([[m[0], m[1], d] for m, d in cands], dtype=np.int32).reshape(-1)
    s0, s1 = ann.tensor_shape
    g0, g1 = ann.granularity
    _device.check(_lib.load().pit_cover_counts(packed.data_ptr(), s0, s1, g0, g1, len(cands), flat.ctypes.data,
                                               occ.data_ptr(), ws, out.data_ptr(), _device.stream_ptr()),
                  IndexBuildError)
    host = out.cpu().numpy().astype(np.int64)
    res, off = [], 0
    for ng, _, _ in geo:
        res.append(host[off : off + ng])
        off += ng
    return res
