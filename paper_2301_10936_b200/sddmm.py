"""Output-sparse matmul (SDDMM): C = A . B only inside the live micro-tiles of C's annotation.

SURVEY 8(f)3. The reference documents the output-side plan as the mirror of pit:m and leaves it
unwired (pkg/README.md:150-153 "The matmul n-axis plan ... is not wired up"), so this
module extends the operator surface in the reference's own terms: a ``SparsityAnnotation`` on the
*output*, the engine's layout contract (the operand on the permuted axis is the contiguous one:
B column-major, the mirror of pit:m's row-major A; never converted silently -> ``LayoutError``),
``ExecError`` for bad shapes. Uses: attention scores S = Q.K^T inside the block mask (C3's
producer side), and the ReLU-masked activation gradient dH = (dY . W2^T) * 1[H > 0] (C4 backward).

Semantics: every element of a live micro-tile of C is written with (A . B)[i, j] (rounded once
from fp32 to the operand dtype); elements of dead micro-tiles are never written, so ``out``
keeps what it held (the default ``out`` is zeros, i.e. the masked product). With ``gate``, a
stored element is zeroed where gate <= 0.

Execution: csrc/pit_sddmm.cu (tcgen05, TMA): two indexes of the output annotation from the K1
detection kernels — units of (128 rows x up to four live 64-column blocks) and the fine
occupancy bitmap that predicates the epilogue's 16-byte stores. bf16 / fp16 only.
"""

from __future__ import annotations

import ctypes as C

from . import _device, _lib
from .executor import DenseTensor, ExecError, LayoutError, _is_torch, _torch_layout
from .index import build_index, build_occupancy
from .sparsity import SparsityAnnotation
from .tiles import COL_MAJOR, ROW_MAJOR

UNIT_MICRO = (128, 64)


def _as_tensor(x):
    return x.array if isinstance(x, DenseTensor) else x


def output_indexes(ann: SparsityAnnotation):
    """(unit index at micro (128, 64), occupancy bitmap at the annotation granularity), both with the
    column axis permuted, from one annotation (device or host bits): two detection launches and one
    compaction."""
    return build_index(ann, UNIT_MICRO, "k"), build_occupancy(ann, ann.granularity, "k")


def output_indexes_from_tensor(values, granularity):
    """The two output indexes straight from the values of a tensor shaped like C (live micro-tile =
    any element != 0): e.g. dH's mask is H's own (1, 32) activation pattern. Everything stays on the
    device (K1 detection twice + compaction), so the call is CUDA-graph capturable -- unlike
    ``from_mask`` on a CUDA tensor, which returns host bits."""
    from .index import build_index_from_tensor

    gran = (int(granularity[0]), int(granularity[1]))
    fine = build_index_from_tensor(values, gran, "k")
    return build_index_from_tensor(values, UNIT_MICRO, "k"), fine.occupancy_words()


class _OutputSpec:
    """Shape and micro-tile of C when its indexes come from values (no annotation object)."""

    def __init__(self, shape, granularity):
        self.tensor_shape = tuple(int(d) for d in shape)
        self.granularity = tuple(int(g) for g in granularity)


def run_sddmm_like(A, B, like, granularity, out=None, gate=None) -> DenseTensor:
    """``run_sddmm`` with C's live micro-tiles detected on the device from ``like`` (a CUDA tensor
    shaped like C): the ReLU-masked activation gradient dH = (dY . W2^T) * 1[H > 0] inside H's
    live 1x32 micro-tiles is ``run_sddmm_like(dY, W2.t(), H, (1, 32), gate=H)``."""
    like = _as_tensor(like)
    if not (_is_torch(like) and like.is_cuda and like.dim() == 2):
        raise ExecError("like must be a 2-D CUDA tensor shaped like the output")
    spec = _OutputSpec(like.shape, granularity)
    return run_sddmm(A, B, spec, out=out, gate=gate, indexes=output_indexes_from_tensor(like, granularity))


def _launch(A2, Bt2, C2, M, N, K, batch, ann, gate, indexes):
    torch = __import__("torch")
    if A2.dtype not in (torch.bfloat16, torch.float16):
        raise ExecError(f"output-sparse plan runs on bf16 / fp16 operands, got {A2.dtype}")
    if Bt2.dtype != A2.dtype or C2.dtype != A2.dtype:
        raise ExecError("dtype mismatch between operands")
    g0, g1 = (int(g) for g in ann.granularity)
    if g1 % 8:
        raise ExecError(f"output micro-tile width {g1} must be a multiple of 8 columns")
    uidx, occ = indexes if indexes is not None else output_indexes(ann)
    uc, us, keep_u = uidx.device_ptrs()
    a = _lib.SddmmArgs()
    a.dtype = _device.dtype_code(A2)
    a.A, a.lda = A2.data_ptr(), A2.stride(0)
    a.B, a.ldb = Bt2.data_ptr(), Bt2.stride(0)
    a.C, a.ldc = C2.data_ptr(), C2.stride(0)
    a.M, a.N, a.K, a.batch = M, N, K, batch
    a.unit_counts, a.unit_slots = uc, us
    a.unit_slot_stride, a.n_unit_groups = uidx.pit_grid, uidx.n_groups
    a.occ, a.words_per_group = occ.data_ptr(), occ.shape[1]
    a.g0, a.g1 = g0, g1
    if gate is not None:
        gate = gate.array if isinstance(gate, DenseTensor) else gate
        if tuple(gate.shape) != tuple(C2.shape) or gate.dtype != C2.dtype or gate.stride(1) != 1:
            raise ExecError("gate must be a row-major tensor shaped and typed like the output")
        a.gate, a.ldgate = gate.data_ptr(), gate.stride(0)
    lib = _lib.load()
    ws = torch.empty(max(int(lib.pit_sddmm_workspace_bytes(C.byref(a))), 4), dtype=torch.uint8, device=A2.device)
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    _device.check(lib.pit_sddmm(C.byref(a), _device.stream_ptr()), ExecError)
    return keep_u, occ, ws


def run_sddmm(A, B, ann: SparsityAnnotation, out=None, gate=None, indexes=None) -> DenseTensor:
    """C[M, N] = A[M, K] . B[K, N] inside the live micro-tiles of ``ann`` (annotation of C).

    A row-major, B column-major (B^T row-major storage), CUDA tensors or DenseTensors thereof.
    ``out``: optional [M, N] row-major tensor written in place (dead micro-tiles untouched);
    ``indexes``: optional precomputed ``output_indexes(ann)`` (e.g. inside a CUDA graph)."""
    torch = __import__("torch")
    At, Bt = _as_tensor(A), _as_tensor(B)
    if not (_is_torch(At) and _is_torch(Bt) and At.is_cuda and Bt.is_cuda):
        raise ExecError("the output-sparse plan takes CUDA tensors")
    if At.dim() != 2 or Bt.dim() != 2:
        raise ExecError("shape mismatch: expected 2-D operands")
    M, K = (int(d) for d in At.shape)
    K2, N = (int(d) for d in Bt.shape)
    if K != K2:
        raise ExecError(f"shape mismatch: A {tuple(At.shape)} vs B {tuple(Bt.shape)}")
    if tuple(ann.tensor_shape) != (M, N):
        raise ExecError(f"annotation shape {tuple(ann.tensor_shape)} does not match the output {(M, N)}")
    if _torch_layout(At) != ROW_MAJOR:
        raise LayoutError("output-sparse plan requires A in row_major")
    if _torch_layout(Bt) != COL_MAJOR and not (N == 1 or K == 1):
        raise LayoutError("output-sparse plan requires B in col_major (the mirror of pit:m's row-major A)")
    if out is None:
        out = torch.zeros((M, N), dtype=At.dtype, device=At.device)
    else:
        out = _as_tensor(out)
        if tuple(out.shape) != (M, N) or _torch_layout(out) != ROW_MAJOR:
            raise ExecError("out must be a row-major [M, N] tensor")
    _launch(At, Bt.t(), out, M, N, K, 1, ann, gate, indexes)
    return DenseTensor(out)


def run_batched_sddmm(A3, B3, ann: SparsityAnnotation, out=None, gate=None, indexes=None):
    """Per-slice output-sparse products in one launch (prevalent axis = batch / heads).

    A3 [b, M, K] row-major contiguous; B3 [b, K, N] column-major per slice (i.e. B3.transpose(1, 2)
    contiguous, e.g. the keys K[b, N, 64] of an attention head viewed as K^T); ``ann`` annotates the
    slices stacked along rows, shape [b*M, N]. Returns out [b, M, N]."""
    torch = __import__("torch")
    if not (_is_torch(A3) and _is_torch(B3) and A3.is_cuda and B3.is_cuda):
        raise ExecError("the output-sparse plan takes CUDA tensors")
    if A3.dim() != 3 or B3.dim() != 3:
        raise ExecError("batched operands must have rank 3")
    b, M, K = (int(d) for d in A3.shape)
    b2, K2, N = (int(d) for d in B3.shape)
    if b != b2 or K != K2:
        raise ExecError(f"shape mismatch: A {tuple(A3.shape)} vs B {tuple(B3.shape)}")
    if tuple(ann.tensor_shape) != (b * M, N):
        raise ExecError(f"annotation shape {tuple(ann.tensor_shape)} does not match the stacked output {(b * M, N)}")
    if not A3.is_contiguous():
        raise LayoutError("output-sparse plan requires A slices row_major and stacked")
    Bt3 = B3.transpose(1, 2)
    if not Bt3.is_contiguous():
        raise LayoutError("output-sparse plan requires B slices in col_major, stacked")
    if b > 1 and M % 128:
        raise ExecError("batched output-sparse plan needs M to be a multiple of 128")
    if out is None:
        out = torch.zeros((b, M, N), dtype=A3.dtype, device=A3.device)
    elif tuple(out.shape) != (b, M, N) or not out.is_contiguous():
        raise ExecError("out must be a contiguous [b, M, N] tensor")
    g = gate.reshape(b * M, N) if gate is not None else None
    _launch(A3.reshape(b * M, K), Bt3.reshape(b * N, K), out.view(b * M, N), M, N, K, b, ann, g, indexes)
    return out
