"""Sparse operator execution on B200: SRead -> tensor-core tile compute -> SWrite.

Mirrors the operator surface of ``pittile.executor`` (reference pkg/src/pittile/executor.py:
``sread`` :170-208, ``swrite`` :211-264, ``run_matmul_with_index`` :464-516,
``run_sparse_matmul`` :519-537) with the same validation order, error types and messages.
Execution is one launch of a fused kernel from libpit_b200.so:

* bf16 / fp16 operands -> tcgen05 kernels (``pit:k`` gathered-K: cp.async row gathers, TMA boxes
  for runs of consecutive live k; ``pit:m`` and dense as union-row tiles on CTA pairs);
* fp32 / f64 operands -> CUDA-core FFMA / DFMA kernels (the reference's f32/f64 dtypes,
  executor.py:40-41; TF32 is never used, so fp32 parity holds at 1e-5).

Host numpy operands are uploaded through pinned staging and the result is read back, so the
reference's numpy-in / numpy-out contract holds; CUDA tensors stay on the device end to end.
There is no CPU fallback: without a GPU every call raises.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Union

import numpy as np

from . import _device, _lib
from .index import PIT_DIMS, MicroTileIndex, build_index
from .policy import SparseKernelPlan, dense_launches, launches_from_counts
from .sparsity import SparsityAnnotation
from .tiles import COL_MAJOR, ROW_MAJOR


class ExecError(ValueError):
    pass


class LayoutError(ExecError):
    pass


_NP_DTYPES = (np.dtype(np.float32), np.dtype(np.float64))
_MAGIC = b"PITT"
_CODES = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}
_FROM_CODE = {v: k for k, v in _CODES.items()}


def _torch():
    import torch

    return torch


def _is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _torch_layout(t) -> Optional[str]:
    if t.dim() != 2:
        return ROW_MAJOR if t.is_contiguous() else None
    s0, s1 = t.stride()
    r, c = t.shape
    if (s1 == 1 or c == 1) and (s0 == c or r == 1):
        return ROW_MAJOR
    if (s0 == 1 or r == 1) and (s1 == r or c == 1):
        return COL_MAJOR
    return None


@dataclass
class DenseTensor:
    """Contiguous 2-D (or n-d) buffer; ``array`` is a numpy array (host) or a torch tensor."""

    array: object

    def __post_init__(self):
        if _is_torch(self.array):
            torch = _torch()
            if self.array.dtype not in (torch.float32, torch.float64, torch.bfloat16, torch.float16):
                raise ExecError(f"unsupported dtype {self.array.dtype}")
            if _torch_layout(self.array) is None:
                raise ExecError("tensor buffer must be contiguous")
            return
        if self.array.dtype not in _NP_DTYPES:
            raise ExecError(f"unsupported dtype {self.array.dtype}")
        if not (self.array.flags.c_contiguous or self.array.flags.f_contiguous):
            raise ExecError("tensor buffer must be contiguous")

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(self.array.shape)

    @property
    def dtype(self):
        return self.array.dtype

    @property
    def is_device(self) -> bool:
        return _is_torch(self.array) and self.array.is_cuda

    @property
    def layout(self) -> str:
        if _is_torch(self.array):
            return _torch_layout(self.array)
        return ROW_MAJOR if self.array.flags.c_contiguous else COL_MAJOR

    def numpy(self) -> np.ndarray:
        return _device.to_host(self.array, self.layout) if _is_torch(self.array) else self.array

    @classmethod
    def from_array(cls, arr, layout: str = ROW_MAJOR, dtype=None) -> "DenseTensor":
        if _is_torch(arr):
            t = arr if dtype is None else arr.to(dtype)
            t = t.contiguous() if layout == ROW_MAJOR else t.t().contiguous().t()
            return cls(t)
        a = np.asarray(arr, dtype=dtype)
        if a.dtype not in _NP_DTYPES:
            a = a.astype(np.float32)
        return cls(np.array(a, order="C" if layout == ROW_MAJOR else "F", copy=True))

    @classmethod
    def zeros(cls, shape, dtype=np.float32, layout: str = ROW_MAJOR) -> "DenseTensor":
        return cls(np.zeros(shape, dtype=dtype, order="C" if layout == ROW_MAJOR else "F"))


def convert_layout(t: DenseTensor, layout: str) -> DenseTensor:
    """Copy into the requested memory order (explicit only; executor.py:79-89)."""
    if layout not in (ROW_MAJOR, COL_MAJOR):
        raise LayoutError(f"unknown layout {layout!r}")
    if t.layout == layout:
        return t
    return DenseTensor.from_array(t.array, layout=layout)


def save_tensor(t: DenseTensor, path: Union[str, Path]) -> None:
    """``PITT`` binary: 16-byte header, int64 extents, raw little-endian values in memory order."""
    arr = t.numpy()
    if arr.dtype not in _CODES:
        arr = arr.astype(np.float32)
    col = t.layout == COL_MAJOR
    header = _MAGIC + struct.pack("<BBB9x", _CODES[arr.dtype], arr.ndim, 1 if col else 0)
    body = np.ascontiguousarray(arr.ravel(order="F" if col else "C")).astype(arr.dtype.newbyteorder("<"))
    Path(path).write_bytes(header + struct.pack(f"<{arr.ndim}q", *arr.shape) + body.tobytes())


def load_tensor(path: Union[str, Path]) -> DenseTensor:
    raw = Path(path).read_bytes()
    if len(raw) < 16 or raw[:4] != _MAGIC:
        raise ExecError(f"{path}: not a tensor file (bad magic)")
    code, rank, lay = struct.unpack("<BBB9x", raw[4:16])
    if code not in _FROM_CODE:
        raise ExecError(f"{path}: unknown dtype code {code}")
    shape = struct.unpack(f"<{rank}q", raw[16 : 16 + 8 * rank])
    dt = _FROM_CODE[code]
    vals = np.frombuffer(raw[16 + 8 * rank :], dtype=dt.newbyteorder("<"), count=int(np.prod(shape)))
    order = "F" if lay == 1 else "C"
    return DenseTensor(np.array(vals.astype(dt).reshape(shape, order=order), order=order, copy=True))


@dataclass(frozen=True)
class Permutation:
    axis: str
    mapping: np.ndarray

    def __post_init__(self):
        m = np.asarray(self.mapping, dtype=np.int64)
        object.__setattr__(self, "mapping", m)
        if m.ndim != 1 or not np.array_equal(np.sort(m), np.arange(m.size)):
            raise ExecError(f"mapping is not a bijection on [0,{m.size})")

    @property
    def extent(self) -> int:
        return int(self.mapping.size)


def invert(p: Permutation) -> Permutation:
    inv = np.empty_like(p.mapping)
    inv[p.mapping] = np.arange(p.mapping.size)
    return Permutation(p.axis, inv)


def apply_permutation(t, p: Permutation, dim: Optional[int] = None):
    """out[..., mapping[i], ...] = in[..., i, ...] (a test utility for invariance checks)."""
    is_dt = isinstance(t, DenseTensor)
    arr = t.numpy() if is_dt else np.asarray(t)
    if dim is None:
        if p.axis not in PIT_DIMS:
            raise ExecError(f"cannot infer dimension for axis {p.axis!r}; pass dim")
        dim = PIT_DIMS[p.axis]
    if arr.shape[dim] != p.extent:
        raise ExecError(f"extent {arr.shape[dim]} does not match permutation {p.extent}")
    out = np.empty_like(arr)
    sel = [slice(None)] * arr.ndim
    sel[dim] = p.mapping
    out[tuple(sel)] = arr
    return DenseTensor.from_array(out, layout=t.layout, dtype=arr.dtype) if is_dt else out


@dataclass
class ExecStats:
    launches: int = 0
    gathered_micro_tiles: int = 0


def _array(x):
    return x.array if isinstance(x, DenseTensor) else (x if _is_torch(x) else np.asarray(x))


# ---------------------------------------------------------------------------- SRead / SWrite
def _gather_checks(arr_shape, idx: MicroTileIndex, group: int, n_slots: int, start: int, for_write: bool):
    t0, t1 = idx.micro_tile
    d = idx.pit_dim
    if group < 0 or group >= idx.n_groups:
        raise ExecError(f"group {group} out of range [0,{idx.n_groups})")
    t_d, t_o = (t0, t1) if d == 0 else (t1, t0)
    coords = idx.group(group)[start : start + n_slots]
    off_o = group * t_o
    v_o = min(t_o, arr_shape[1 - d] - off_o)
    if (for_write and v_o <= 0) or (not for_write and off_o >= arr_shape[1 - d]):
        raise ExecError(f"group {group} window outside tensor")
    if coords.size and int(coords.max()) * t_d >= arr_shape[d]:
        raise ExecError("micro-tile coordinate out of range")
    edge = bool(coords.size) and (int(coords.max()) + 1) * t_d > arr_shape[d]
    return coords, t_d, v_o, edge


def _tensor_geometry(t):
    """(ld, col_major) of a 2-D device tensor."""
    s0, s1 = t.stride()
    if _torch_layout(t) == COL_MAJOR and t.shape[0] > 1:
        return s1, 1
    return s0, 0


def sread(src, idx: MicroTileIndex, group: int, tile_buffer, start: int = 0) -> int:
    """Gather one group's micro-tiles (stored order) into consecutive tile slots; see executor.py:170."""
    arr = _array(src)
    d = idx.pit_dim
    t_d = idx.micro_tile[0] if d == 0 else idx.micro_tile[1]
    n_slots = tile_buffer.shape[d] // t_d
    coords, t_d, v_o, edge = _gather_checks(arr.shape, idx, group, n_slots, start, False)
    full = coords.size == n_slots and v_o == tile_buffer.shape[1 - d]
    torch = _torch()
    dev = _device.require_cuda()
    x = _device.to_device(arr)
    host_tile = not _is_torch(tile_buffer)
    tile = _device.to_device(np.ascontiguousarray(tile_buffer)) if host_tile else tile_buffer
    if not tile.is_contiguous():
        raise ExecError("tile buffer must be contiguous")
    user_tile = tile
    if tile.dtype != x.dtype:
        # the C ABI types the tile with the tensor's dtype: gather into a tile of that dtype and
        # cast on the way back (numpy assignment semantics, executor.py:205-207)
        tile = tile.to(x.dtype)
    cd = torch.from_numpy(np.ascontiguousarray(coords, dtype=np.int32)).to(dev)
    ld, col = _tensor_geometry(x)
    lib = _lib.load()
    _device.check(lib.pit_sread(x.data_ptr(), _device.dtype_code(x), arr.shape[0], arr.shape[1], ld, col,
                                tile.data_ptr(), tile.shape[0], tile.shape[1], idx.micro_tile[0], idx.micro_tile[1],
                                d, group, cd.data_ptr(), coords.size, int((not full) or edge),
                                _device.stream_ptr()), ExecError)
    if host_tile:
        tile_buffer[...] = _device.to_host(tile)
    elif tile is not user_tile:
        user_tile.copy_(tile)
    return int(coords.size)


def swrite(tile_buffer, dst, idx: MicroTileIndex, group: int, start: int = 0, accumulate: bool = False) -> int:
    """Scatter tile slots back to their micro-tiles (mirror of sread; executor.py:211-264)."""
    is_dt = isinstance(dst, DenseTensor)
    arr = _array(dst)
    d = idx.pit_dim
    t_d = idx.micro_tile[0] if d == 0 else idx.micro_tile[1]
    n_slots = tile_buffer.shape[d] // t_d
    coords, _, _, _ = _gather_checks(arr.shape, idx, group, n_slots, start, True)
    torch = _torch()
    dev = _device.require_cuda()
    host_dst = not _is_torch(arr)
    x = _device.to_device(arr)
    tile = _device.to_device(np.ascontiguousarray(tile_buffer)) if not _is_torch(tile_buffer) else tile_buffer
    if tile.dtype != x.dtype or not tile.is_contiguous():
        tile = tile.to(x.dtype).contiguous()  # read with the tensor's element size (C ABI contract)
    cd = torch.from_numpy(np.ascontiguousarray(coords, dtype=np.int32)).to(dev)
    ld, col = _tensor_geometry(x)
    lib = _lib.load()
    _device.check(lib.pit_swrite(tile.data_ptr(), x.data_ptr(), _device.dtype_code(x), arr.shape[0], arr.shape[1], ld,
                                 col, tile.shape[0], tile.shape[1], idx.micro_tile[0], idx.micro_tile[1], d, group,
                                 cd.data_ptr(), coords.size, int(bool(accumulate)), _device.stream_ptr()), ExecError)
    if host_dst:
        arr[...] = _device.to_host(x, COL_MAJOR if arr.flags.f_contiguous and not arr.flags.c_contiguous else ROW_MAJOR)
    elif is_dt:
        pass
    return int(coords.size)


# ------------------------------------------------------------------------------ verification
def run_dense_reference(a, b) -> np.ndarray:
    """f64 oracle, reduction ascending, multiply then add — the scalar triple loop's exact
    operation sequence (executor.py:267-283), computed on the GPU without FMA contraction."""
    A = _array(a)
    B = _array(b)
    if len(A.shape) != 2 or len(B.shape) != 2 or A.shape[1] != B.shape[0]:
        raise ExecError(f"shape mismatch {tuple(A.shape)} @ {tuple(B.shape)}")
    torch = _torch()
    dev = _device.require_cuda()
    Ad = _device.to_device(np.asarray(A, dtype=np.float64) if not _is_torch(A) else A).to(torch.float64)
    Bd = _device.to_device(np.asarray(B, dtype=np.float64) if not _is_torch(B) else B).to(torch.float64).contiguous()
    m, k = Ad.shape
    n = Bd.shape[1]
    Cd = torch.empty((m, n), dtype=torch.float64, device=dev)
    if m and n:
        lib = _lib.load()
        s0, s1 = Ad.stride()
        _device.check(lib.pit_dense_reference_f64(Ad.data_ptr(), s0, s1, Bd.data_ptr(), Bd.stride(0), Cd.data_ptr(),
                                                  m, n, k, _device.stream_ptr()), ExecError)
    return _device.to_host(Cd)


def max_rel_error(result, oracle, floor: float = 1e-6) -> float:
    """Normwise relative error: peak |x - y| over peak |y| (floored), executor.py:294-300."""
    x = _host64(result)
    y = _host64(oracle)
    if not y.size:
        return 0.0
    return float(np.max(np.abs(x - y))) / max(float(np.max(np.abs(y))), floor)


def verify_close(result, oracle, rtol: float = 1e-5, atol: float = 1e-6) -> bool:
    x = _host64(result)
    y = _host64(oracle)
    if not y.size:
        return True
    return bool(np.max(np.abs(x - y)) <= atol + rtol * float(np.max(np.abs(y))))


def _host64(x) -> np.ndarray:
    if isinstance(x, DenseTensor):
        x = x.numpy()
    elif _is_torch(x):
        x = _device.to_host(x)
    return np.asarray(x, dtype=np.float64)


# ---------------------------------------------------------------------------------- matmul
def _check_matmul_operands(plan: SparseKernelPlan, A: DenseTensor, B: DenseTensor) -> None:
    if len(A.shape) != 2 or len(B.shape) != 2 or A.shape[1] != B.shape[0]:
        raise ExecError(f"shape mismatch {A.shape} @ {B.shape}")
    if A.dtype != B.dtype:
        raise ExecError(f"mixed dtypes {A.dtype} and {B.dtype}")
    ext = plan.extents
    if (ext["m"], ext["k"]) != A.shape or ext["n"] != B.shape[1]:
        raise ExecError(f"plan bound to {dict(ext)} but got A{A.shape} B{B.shape}")
    if not plan.is_dense and A.layout != plan.sparse_layout:
        # a degenerate extent is both layouts at once
        if not (A.shape[0] == 1 or A.shape[1] == 1):
            raise LayoutError(
                f"plan requires the sparse operand in {plan.sparse_layout}, got {A.layout}; use convert_layout first"
            )


_PLAN_CODE = {"dense": _lib.PIT_PLAN_DENSE, "m": _lib.PIT_PLAN_PIT_M, "k": _lib.PIT_PLAN_PIT_K}


def _attach_workspace(a, keep) -> None:
    """Caller-owned scratch for pit_spmm (split gathered-K units): a stream-ordered torch allocation
    per call, so concurrent streams never share it and CUDA-graph capture draws it from the graph's
    pool."""
    n = int(_lib.load().pit_spmm_workspace_bytes(C.byref(a)))
    if n > 0:
        buf = _torch().empty(n, dtype=_torch().uint8, device=_device.require_cuda())
        a.workspace, a.workspace_bytes = buf.data_ptr(), n
        keep.append(buf)


def spmm_device(plan: SparseKernelPlan, Ad, Bd, idx: Optional[MicroTileIndex], out=None, force_simt: bool = False):
    """Launch the fused SpMM on device tensors (no validation beyond the C ABI's); returns C."""
    torch = _torch()
    dev = _device.require_cuda()
    M, K = int(Ad.shape[0]), int(Ad.shape[1])
    N = int(Bd.shape[1])
    if (Bd.stride(1) != 1 and N > 1) or (Bd.stride(0) * Bd.element_size()) % 16:
        Bd = Bd.contiguous()  # pitched row-major views (column slabs) are used as they are
    C_ = out if out is not None else torch.empty((M, N), dtype=Ad.dtype, device=dev)
    a = _lib.SpmmArgs()
    a.plan = _PLAN_CODE["dense" if plan.is_dense else plan.pit_axis]
    a.dtype = _device.dtype_code(Ad)
    a.M, a.N, a.K = M, N, K
    a.A = Ad.data_ptr()
    a.sam, a.sak = Ad.stride()
    if M == 1:
        a.sam = 1 if plan.pit_axis == "k" else a.sam
    if K == 1:
        a.sak = 1 if plan.pit_axis != "k" else a.sak
    a.B = Bd.data_ptr()
    a.ldb = Bd.stride(0) if N > 1 or K > 1 else N
    a.C = C_.data_ptr()
    a.ldc = C_.stride(0)
    keep = []
    if not plan.is_dense:
        t0, t1 = idx.micro_tile
        a.t0, a.t1 = t0, t1
        a.n_groups = idx.n_groups
        a.slot_stride = idx.pit_grid
        if plan.pit_axis == "k":
            a.counts, a.slots, alive = idx.device_ptrs()
            keep += list(alive)
        else:
            occ = idx.occupancy_words()
            rows, n_rows = idx.union_coords()
            keep += [occ, rows, n_rows]
            a.counts, _, alive = idx.device_ptrs()  # live rows per K-group (globally dead K-blocks)
            keep += list(alive)
            a.occ = occ.data_ptr()
            a.words_per_group = occ.shape[1]
            a.rows, a.n_rows = rows.data_ptr(), n_rows.data_ptr()
            a.n_rows_bound = M
    a.force_simt = int(force_simt)
    _attach_workspace(a, keep)
    lib = _lib.load()
    _device.check(lib.pit_spmm(C.byref(a), _device.stream_ptr()), ExecError)
    return C_


def run_matmul_with_index(
    plan: SparseKernelPlan,
    A: DenseTensor,
    B: DenseTensor,
    idx: Optional[MicroTileIndex],
    workers: int = 1,
    stats: Optional[ExecStats] = None,
) -> DenseTensor:
    """Run a matmul plan against a prebuilt index (ignored for the dense plan)."""
    _check_matmul_operands(plan, A, B)
    if plan.op_kind != "matmul":
        raise ExecError(f"not a matmul plan: {plan.op_kind}")
    if not plan.is_dense:
        if idx is None:
            raise ExecError("sparse plan needs a micro-tile index")
        if idx.pit_axis != plan.pit_axis or tuple(idx.micro_tile) != tuple(plan.micro_tile):
            raise ExecError(
                f"index ({idx.pit_axis}, {idx.micro_tile}) does not match plan ({plan.pit_axis}, {plan.micro_tile})"
            )
        if plan.pit_axis not in ("m", "k"):
            raise ExecError(f"matmul axis {plan.pit_axis!r} is not executable (m and k only)")
        dim = PIT_DIMS[plan.pit_axis]
        t = plan.micro_tile
        want_groups = -(-A.shape[1 - dim] // t[1 - dim])
        if idx.n_groups != want_groups:
            raise ExecError(f"index has {idx.n_groups} groups, operand needs {want_groups}")
    host = not (A.is_device and B.is_device)
    if host and _pipelined_ok(A, B):
        Cres = _run_host_pipelined(plan, A, B, idx)
    elif host and _stageable(B):
        # large host B that is numpy or pageable (the reference's own contract): one copy into pinned
        # memory, then the same pipelined path (B slab uploads, per-slab SpMM and C slab downloads
        # overlap); C comes back as numpy when B came in as numpy (a view of the pinned result)
        Bp = _torch().from_numpy(np.ascontiguousarray(B.array)) if not _is_torch(B.array) else B.array.contiguous()
        Cres = _run_host_pipelined(plan, A, DenseTensor(Bp.pin_memory()), idx)
        if not _is_torch(B.array):
            Cres = Cres.numpy()
    else:
        Ad = _device.to_device(A.array)
        Bd = _device.to_device(B.array)
        Cd = spmm_device(plan, Ad, Bd, idx)
        Cres = _device.to_host(Cd) if host else Cd
    if stats is not None:
        if plan.is_dense:
            stats.launches += dense_launches(plan)
        else:
            stats.launches += launches_from_counts(plan, idx.counts)
            stats.gathered_micro_tiles += idx.total
    return DenseTensor(Cres)


# host-buffer path: B column slabs upload, per-slab SpMM and C slab download run on three streams
_PIPE_MIN_BYTES = 32 << 20
_pipe_streams = {}


def _pipelined_ok(A: DenseTensor, B: DenseTensor) -> bool:
    """Large host-resident B (pinned torch tensor): overlap PCIe with compute."""
    b = B.array
    return (_is_torch(b) and not b.is_cuda and b.is_pinned() and _torch_layout(b) == ROW_MAJOR
            and b.numel() * b.element_size() >= _PIPE_MIN_BYTES and b.shape[1] >= 1024)


def _stageable(B: DenseTensor) -> bool:
    """Large row-major host B that is not pinned (numpy, pageable torch): worth one pinned copy."""
    b = B.array
    if _is_torch(b):
        if b.is_cuda or b.is_pinned():
            return False
        n_bytes, layout, ndim = b.numel() * b.element_size(), _torch_layout(b), b.dim()
    else:
        b = np.asarray(b)
        n_bytes, ndim = b.nbytes, b.ndim
        layout = ROW_MAJOR if b.flags.c_contiguous else COL_MAJOR
    return ndim == 2 and layout == ROW_MAJOR and n_bytes >= _PIPE_MIN_BYTES and b.shape[1] >= 1024


def _slab_schedule(N: int):
    """(first column, width) of the B / C column slabs. Small slabs at both ends: the first one
    starts the C downloads early, the last one keeps the tail (its SpMM and download) short; wide
    ones in the middle copy in longer rows, which PCIe moves faster while both directions are busy.
    1/16, 3/16, 1/4, 1/4, 3/16, 1/16 of N measured 2-3% faster than eight equal slabs
    (scripts/e2e_timeline.py, 8192^3: 6.34 -> 6.19 ms). Widths are multiples of 256 columns."""
    if N < 4096:
        slab = max(1024, -(-(-(-N // 8)) // 256) * 256)
        return [(j0, min(slab, N - j0)) for j0 in range(0, N, slab)]
    cuts = sorted({0, N} | {round(N * c / 16 / 256) * 256 for c in (1, 4, 8, 12, 15)})
    return [(a, b - a) for a, b in zip(cuts, cuts[1:])]


def _run_host_pipelined(plan: SparseKernelPlan, A: DenseTensor, B: DenseTensor, idx):
    torch = _torch()
    dev = _device.require_cuda()
    lib = _lib.load()
    main = torch.cuda.current_stream()
    if dev.index not in _pipe_streams:
        _pipe_streams[dev.index] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    s_up, s_down = _pipe_streams[dev.index]
    Ad = _device.to_device(A.array)
    Bh = B.array
    K, N = Bh.shape
    M = Ad.shape[0]
    eb = Bh.element_size()
    Bd = torch.empty((K, N), dtype=Bh.dtype, device=dev)
    Cd = torch.empty((M, N), dtype=Bh.dtype, device=dev)
    Ch = torch.empty((M, N), dtype=Bh.dtype, pin_memory=True)
    up_done = []
    s_up.wait_stream(main)
    for j0, w in _slab_schedule(N):
        with torch.cuda.stream(s_up):
            _device.check(lib.pit_copy2d_async(Bd.data_ptr() + j0 * eb, N * eb, Bh.data_ptr() + j0 * eb, N * eb,
                                               w * eb, K, s_up.cuda_stream))
            ev = torch.cuda.Event()
            ev.record(s_up)
        up_done.append((j0, w, ev))
    for j0, w, ev in up_done:
        main.wait_event(ev)
        spmm_device(plan, Ad, Bd[:, j0 : j0 + w], idx, out=Cd[:, j0 : j0 + w])
        ev_c = torch.cuda.Event()
        ev_c.record(main)
        s_down.wait_event(ev_c)
        with torch.cuda.stream(s_down):
            _device.check(lib.pit_copy2d_async(Ch.data_ptr() + j0 * eb, N * eb, Cd.data_ptr() + j0 * eb, N * eb,
                                               w * eb, M, s_down.cuda_stream))
    main.wait_stream(s_down)
    for t in (Bd, Cd):
        t.record_stream(s_up)
        t.record_stream(s_down)
    main.synchronize()
    return Ch


def run_sparse_matmul(
    plan: SparseKernelPlan,
    A: DenseTensor,
    B: DenseTensor,
    ann: Optional[SparsityAnnotation],
    workers: int = 1,
    stats: Optional[ExecStats] = None,
) -> DenseTensor:
    """Detect, index and execute in one call (executor.py:519-537)."""
    _check_matmul_operands(plan, A, B)
    idx = None
    if not plan.is_dense:
        if ann is None:
            raise ExecError("sparse plan needs a sparsity annotation")
        if tuple(ann.tensor_shape) != A.shape:
            raise ExecError(f"annotation {ann.tensor_shape} does not describe A {A.shape}")
        idx = build_index(ann, plan.micro_tile, plan.pit_axis, workers=workers)
    return run_matmul_with_index(plan, A, B, idx, workers=workers, stats=stats)


# ------------------------------------------------------------------------------ reduce_sum
def reduce_sum_reference(a) -> np.ndarray:
    """f64 row sums (executor.py:286-291), computed on the GPU."""
    A = _array(a)
    if len(A.shape) != 2:
        raise ExecError("reduce_sum oracle expects rank 2")
    torch = _torch()
    Ad = _device.to_device(np.asarray(A, dtype=np.float64) if not _is_torch(A) else A).to(torch.float64).contiguous()
    out = torch.empty(Ad.shape[0], dtype=torch.float64, device=Ad.device)
    lib = _lib.load()
    _device.check(lib.pit_reduce_rows(Ad.data_ptr(), _lib.PIT_F64, Ad.shape[0], Ad.shape[1], Ad.stride(0), None, 0, 0,
                                      1, out.data_ptr(), _device.stream_ptr()), ExecError)
    return _device.to_host(out)


def run_sparse_reduce_sum(
    plan: SparseKernelPlan,
    A: DenseTensor,
    ann: Optional[SparsityAnnotation],
    workers: int = 1,
    stats: Optional[ExecStats] = None,
) -> DenseTensor:
    """Row reduction over live micro-tiles (executor.py:540-613): one GPU pass, a warp per row;
    rows with no survivor stay exactly 0.0."""
    if plan.op_kind != "reduce_sum":
        raise ExecError(f"not a reduce_sum plan: {plan.op_kind}")
    if len(A.shape) != 2:
        raise ExecError("reduce_sum expects a rank-2 operand")
    ext = plan.extents
    if (ext["p"], ext["l"]) != A.shape:
        raise ExecError(f"plan bound to {dict(ext)} but got A{A.shape}")
    torch = _torch()
    host = not A.is_device
    Ad = _device.to_device(A.array)
    if _torch_layout(Ad) != ROW_MAJOR:
        Ad = Ad.contiguous()
    p, l = A.shape
    out = torch.empty(p, dtype=Ad.dtype, device=Ad.device)
    lib = _lib.load()
    idx = None
    if plan.is_dense:
        mode, occ, wg, block = 0, None, 0, 1
    else:
        if ann is None or tuple(ann.tensor_shape) != A.shape:
            raise ExecError("per-row plan needs an annotation matching A")
        idx = build_index(ann, plan.micro_tile, plan.pit_axis, workers=workers)
        occ_t = idx.occupancy_words()
        occ, wg = occ_t.data_ptr(), occ_t.shape[1]
        mode = 1 if plan.pit_axis == "l" else 2
        block = plan.micro_tile[1]
    _device.check(lib.pit_reduce_rows(Ad.data_ptr(), _device.dtype_code(Ad), p, l, Ad.stride(0), occ, wg, mode, block,
                                      out.data_ptr(), _device.stream_ptr()), ExecError)
    if stats is not None:
        if plan.is_dense:
            stats.launches += dense_launches(plan)
        elif plan.pit_axis == "l":
            # executed tile launches: per block of P rows, the longest row's survivor chunks
            # (executor.py:593-608; differs from the cost model's average, policy.py:181-184)
            P, L = plan.tile.tile_shape
            chunks = -(-idx.counts // L)
            stats.launches += int(sum(chunks[i : i + P].max(initial=0) for i in range(0, p, P)))
            stats.gathered_micro_tiles += idx.total
        else:
            stats.launches += launches_from_counts(plan, idx.counts)
            stats.gathered_micro_tiles += idx.total
    return DenseTensor(_device.to_host(out) if host else out)


# ------------------------------------------------------------------------------ single tile
def _scatter_whole(tile, dst, accumulate: bool) -> None:
    """dst (rank 2, device) = / += tile through SWrite with one micro-tile covering all of dst."""
    torch = _torch()
    rows, cols = int(dst.shape[0]), int(dst.shape[1])
    zero = torch.zeros(1, dtype=torch.int32, device=dst.device)
    ld, col = _tensor_geometry(dst)
    _device.check(_lib.load().pit_swrite(tile.contiguous().data_ptr(), dst.data_ptr(), _device.dtype_code(dst), rows,
                                         cols, ld, col, rows, cols, rows, cols, 0, 0, zero.data_ptr(), 1,
                                         int(accumulate), _device.stream_ptr()), ExecError)


def run_tile(desc, inputs, out, scratch=None) -> None:
    """Execute one dense tile (reference tiles.py:119-148) with the sm_100a kernels: matmul and
    reduce_sum accumulate into ``out``, vec_add assigns. Buffers may be host arrays (``out`` is
    updated in place) or CUDA tensors; ``scratch`` (M, N) is reused for the matmul product."""
    from .tiles import TileError

    in_shapes, out_shape = desc.buffer_shapes()
    if len(inputs) != len(in_shapes):
        raise TileError(f"{desc.op_kind} takes {len(in_shapes)} inputs, got {len(inputs)}")
    for buf, want in zip(inputs, in_shapes):
        if tuple(buf.shape) != want:
            raise TileError(f"input shape {tuple(buf.shape)} does not match tile {want}")
    if tuple(out.shape) != out_shape:
        raise TileError(f"output shape {tuple(out.shape)} does not match tile {out_shape}")
    torch = _torch()
    host_out = not _is_torch(out)
    ins = [_device.to_device(np.asarray(x) if not _is_torch(x) else x) for x in inputs]
    o = _device.to_device(np.asarray(out)) if host_out else out
    o2 = o.reshape(out_shape[0], -1) if desc.op_kind == "matmul" else o.reshape(-1, 1)
    if desc.op_kind == "matmul":
        a, b = ins
        m, k, n = desc.tile_shape
        plan = SparseKernelPlan("matmul", "dense", None, desc, 0.0, 0.0, ROW_MAJOR, dict(m=m, k=k, n=n))
        prod = scratch if _is_torch(scratch) and scratch.is_cuda else torch.empty((m, n), dtype=a.dtype, device=a.device)
        spmm_device(plan, a.contiguous(), b.contiguous(), None, out=prod)
        _scatter_whole(prod, o2, True)
    elif desc.op_kind == "reduce_sum":
        a = ins[0].contiguous()
        sums = torch.empty((a.shape[0], 1), dtype=a.dtype, device=a.device)
        _device.check(_lib.load().pit_reduce_rows(a.data_ptr(), _device.dtype_code(a), a.shape[0], a.shape[1],
                                                  a.stride(0), None, 0, 0, 1, sums.data_ptr(), _device.stream_ptr()),
                      ExecError)
        _scatter_whole(sums, o2, True)
    else:
        _scatter_whole(ins[0].reshape(-1, 1), o2, False)
        _scatter_whole(ins[1].reshape(-1, 1), o2, True)
    if host_out:
        out[...] = _device.to_host(o).reshape(out_shape)


# ------------------------------------------------------------------ batched (prevalent axis)
def stack_slices(A3, plan: SparseKernelPlan):
    """Explicit layout conversion for batched products (convert_layout's counterpart): returns the
    [batch, M, K] operand as a device view over ONE buffer with the slices stacked along M, col-major
    for pit:k ([K, batch*M] row-major underneath) and row-major for dense."""
    torch = _torch()
    x = _device.to_device(np.ascontiguousarray(A3) if not _is_torch(A3) else A3)
    if x.dim() != 3:
        raise ExecError(f"batched operand must have rank 3, got {x.dim()}")
    b, m, k = x.shape
    if plan.is_dense or plan.pit_axis == "m":
        return x.contiguous()
    flat = torch.empty((k, b * m), dtype=x.dtype, device=x.device)
    flat.view(k, b, m).copy_(x.permute(2, 0, 1))
    return flat.view(k, b, m).permute(1, 2, 0)


def _stacked_2d(A3, plan: SparseKernelPlan):
    """The [batch*M, K] 2-D view of a stacked batched operand; LayoutError if A3 is not stacked."""
    b, m, k = (int(d) for d in A3.shape)
    s0, s1, s2 = A3.stride()
    if plan.is_dense or plan.pit_axis == "m":
        ok = s2 == 1 and s1 == k and s0 == m * k
        return A3.reshape(b * m, k) if ok or b * m * k == 0 else _layout_error(plan)
    ok = s1 == 1 and s0 == m and s2 == b * m
    if not (ok or b * m * k == 0 or (m == 1 and b == 1)):
        _layout_error(plan)
    return A3.permute(2, 0, 1).reshape(k, b * m).t()


def _layout_error(plan):
    raise LayoutError(f"batched plan requires slices stacked along M in {plan.sparse_layout}; use stack_slices first")


def build_batched_index_from_tensor(A3, micro_tile, pit_axis="k") -> MicroTileIndex:
    """One detection pass over a stacked [batch, M, K] operand (see stack_slices): the index of the
    stacked [batch*M, K] view, i.e. the per-slice indices back to back (slice b owns groups
    [b*M/t0, (b+1)*M/t0))."""
    from .index import build_index_from_tensor

    if int(A3.shape[1]) % int(micro_tile[0]):
        raise ExecError("batched plans need M to be a multiple of the micro-tile height")
    axis = pit_axis if isinstance(pit_axis, str) else ("m" if pit_axis == 0 else "k")
    dummy = SparseKernelPlan("matmul", axis, tuple(micro_tile), None, 0.0, 0.0,
                             COL_MAJOR if axis == "k" else ROW_MAJOR, {})
    return build_index_from_tensor(_stacked_2d(A3, dummy), micro_tile, pit_axis)


def build_batched_index(anns, micro_tile, pit_axis="k") -> MicroTileIndex:
    """Stacked index from one annotation per slice (each slice's block grid must tile M exactly)."""
    from .sparsity import from_bits

    anns = list(anns)
    if not anns:
        raise ExecError("batched index needs at least one annotation")
    shape, gran = tuple(anns[0].tensor_shape), tuple(anns[0].granularity)
    if any(tuple(a.tensor_shape) != shape or tuple(a.granularity) != gran for a in anns):
        raise ExecError("batched annotations must share shape and granularity")
    if shape[0] % gran[0] or shape[0] % int(micro_tile[0]):
        raise ExecError("batched plans need M to be a multiple of the granularity and the micro-tile height")
    stacked = from_bits(np.concatenate([a.bits() for a in anns], axis=0), (len(anns) * shape[0], shape[1]), gran)
    return build_index(stacked, micro_tile, pit_axis)


def run_batched_matmul_with_index(plan: SparseKernelPlan, A3, B3, idx: Optional[MicroTileIndex],
                                  stats: Optional[ExecStats] = None):
    """C[b] = A[b] @ B[b] for every slice in ONE launch, with A stacked along M (stack_slices) and
    idx the stacked index. Same per-slice semantics as run_matmul_with_index (an
    independent index per slice of the prevalent axis). pit:k gathers k per query/row group; pit:m
    runs every row tile over its slice's B and skips K-blocks in which no row of the tile is live
    (bf16/fp16). Returns a [batch, M, N] tensor on the device (or numpy when B3 is a host array)."""
    torch = _torch()
    if plan.op_kind != "matmul":
        raise ExecError(f"not a matmul plan: {plan.op_kind}")
    host = not _is_torch(B3) or not B3.is_cuda
    Ad = _stacked_2d(A3 if _is_torch(A3) and A3.is_cuda else stack_slices(A3, plan), plan)
    Bd = _device.to_device(np.ascontiguousarray(B3) if not _is_torch(B3) else B3)
    batch, M, K = (int(d) for d in A3.shape)
    if Bd.dim() != 3 or int(Bd.shape[0]) != batch or int(Bd.shape[1]) != K:
        raise ExecError(f"shape mismatch {tuple(A3.shape)} @ {tuple(Bd.shape)}")
    N = int(Bd.shape[2])
    if (plan.extents["m"], plan.extents["k"], plan.extents["n"]) != (M, K, N):
        raise ExecError(f"plan bound to {dict(plan.extents)} but got slices {M}x{K}x{N}")
    if Bd.stride(2) != 1 and N > 1:
        Bd = Bd.contiguous()
    if Ad.dtype != Bd.dtype:
        raise ExecError(f"mixed dtypes {Ad.dtype} and {Bd.dtype}")
    C3 = torch.empty((batch, M, N), dtype=Bd.dtype, device=Bd.device)
    a = _lib.SpmmArgs()
    a.plan = _PLAN_CODE["dense" if plan.is_dense else plan.pit_axis]
    a.dtype = _device.dtype_code(Bd)
    a.M, a.N, a.K = M, N, K
    a.A = Ad.data_ptr()
    a.sam, a.sak = Ad.stride()
    a.B = Bd.data_ptr()
    a.ldb = Bd.stride(1)
    a.C = C3.data_ptr()
    a.ldc = N
    a.batch = batch
    a.b_batch_stride = Bd.stride(0)
    keep = []
    if not plan.is_dense:
        if idx is None or idx.pit_axis != plan.pit_axis or tuple(idx.micro_tile) != tuple(plan.micro_tile):
            raise ExecError(f"batched {plan.pit_axis} plan needs the stacked index of its micro-tile")
        want = batch * -(-M // plan.micro_tile[0]) if plan.pit_axis == "k" else -(-K // plan.micro_tile[1])
        if idx.n_groups != want or (plan.pit_axis == "m" and idx.pit_grid != batch * M):
            raise ExecError(f"index has {idx.n_groups} groups, stacked operand needs {want}")
        a.t0, a.t1 = plan.micro_tile
        a.n_groups = idx.n_groups
        a.slot_stride = idx.pit_grid
        if plan.pit_axis == "k":
            a.counts, a.slots, alive = idx.device_ptrs()
            keep += list(alive)
        else:
            occ = idx.occupancy_words()
            keep.append(occ)
            a.occ = occ.data_ptr()
            a.words_per_group = occ.shape[1]
            if batch == 1:  # a single slice runs the 2-D pit:m kernels: union rows + per-group counts
                rows, n_rows = idx.union_coords()
                a.counts, _, alive = idx.device_ptrs()
                keep += [rows, n_rows, *alive]
                a.rows, a.n_rows = rows.data_ptr(), n_rows.data_ptr()
                a.n_rows_bound = M
    _attach_workspace(a, keep)
    _device.check(_lib.load().pit_spmm(C.byref(a), _device.stream_ptr()), ExecError)
    if stats is not None:
        if plan.is_dense:
            stats.launches += batch * dense_launches(plan)
        elif plan.pit_axis == "k":
            stats.launches += launches_from_counts(plan, idx.counts)
            stats.gathered_micro_tiles += idx.total
        else:  # per slice: its rows' share of every K-block group
            occ = idx.occupancy_words().cpu().numpy().view(np.uint32)
            bits = np.unpackbits(occ.view(np.uint8), bitorder="little").reshape(idx.n_groups, -1)[:, : batch * M]
            per_slice = bits.reshape(idx.n_groups, batch, M).sum(axis=2)
            stats.launches += sum(launches_from_counts(plan, per_slice[:, b]) for b in range(batch))
            stats.gathered_micro_tiles += idx.total
    return _device.to_host(C3.reshape(batch * M, N)).reshape(batch, M, N) if host else C3


def run_sparse_batched_matmul(plan: SparseKernelPlan, A3, B3, anns, stats: Optional[ExecStats] = None):
    """Batched run_sparse_matmul: per-slice annotations -> stacked index -> one launch. pit:m slices
    the tensor-core path cannot take in one launch (fp32, or A / B rows not 16-byte aligned) run
    slice by slice through run_sparse_matmul, each with its own index."""
    if plan.pit_axis == "m" and not _batched_pit_m_ok(A3, B3):
        torch = _torch()
        outs = []
        for b, ann in enumerate(anns):
            Ab = A3[b] if _is_torch(A3) else np.ascontiguousarray(A3[b])
            outs.append(run_sparse_matmul(plan, DenseTensor(Ab), DenseTensor(B3[b]), ann, stats=stats).array)
        return torch.stack(outs) if _is_torch(outs[0]) else np.stack(outs)
    idx = None if plan.is_dense else build_batched_index(anns, plan.micro_tile, plan.pit_axis)
    return run_batched_matmul_with_index(plan, A3, B3, idx, stats=stats)


def _batched_pit_m_ok(A3, B3) -> bool:
    """One tensor-core launch takes the stacked pit:m product: bf16 / fp16, A and B rows 16-byte
    aligned (TMA pitches)."""
    if not (_is_torch(B3) and _is_torch(A3)):
        return False
    torch = _torch()
    es = B3.element_size()
    return B3.dtype in (torch.bfloat16, torch.float16) and (B3.shape[2] * es) % 16 == 0 and \
        (B3.stride(0) * es) % 16 == 0 and A3.dim() == 3 and (A3.stride(1) * A3.element_size()) % 16 == 0
