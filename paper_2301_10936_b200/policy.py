"""Plans: (dense tile, PIT axis) pairs and their micro-tiles.

Host-side contract consumed by the executor (reference policy.py:36-184): the micro-tile is the
tile's sparse-operand projection with extent 1 along the PIT axis; ``pit:m`` wants the sparse
operand row-major and ``pit:k`` column-major; ``plan_launches`` is the logical tile-launch count
that ``ExecStats.launches`` must reproduce.

Cover counting (``cover_group_counts``) uses prefix sums over the block grid — an independent
restatement of the detection kernel's occupancy rule, kept host-side for the cost model.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Optional, Sequence, Union

import numpy as np

from .expr import TensorExpr, operator_kind
from .sparsity import SparsityAnnotation
from .tiles import COL_MAJOR, ROW_MAJOR, KernelRegistry, TileKernelDescriptor

DENSE = "dense"
DEFAULT_TILES = {"matmul": (32, 64, 32), "reduce_sum": (16, 64)}
PIT_DIMS = {"m": 0, "p": 0, "k": 1, "l": 1}


class PlanError(ValueError):
    pass


@dataclass(frozen=True)
class SparseKernelPlan:
    op_kind: str
    pit_axis: str
    micro_tile: Optional[tuple[int, int]]
    tile: TileKernelDescriptor
    tile_cost: float
    estimated_cost: float
    sparse_layout: str
    extents: Mapping[str, int]

    @property
    def is_dense(self) -> bool:
        return self.pit_axis == DENSE


def sparse_operand_axes(op_kind: str) -> tuple[str, str]:
    if op_kind == "matmul":
        return ("m", "k")
    if op_kind == "reduce_sum":
        return ("p", "l")
    raise PlanError(f"op kind {op_kind!r} is not plannable (matmul and reduce_sum only)")


def sparse_operand_shape(op_kind: str, extents: Mapping[str, int]) -> tuple[int, int]:
    a0, a1 = sparse_operand_axes(op_kind)
    return (extents[a0], extents[a1])


def get_micro_tile(op_kind: str, tile_shape: Sequence[int], pit_axis: str, sparse_layout: str = ROW_MAJOR):
    shape = tuple(int(d) for d in tile_shape)
    axes = sparse_operand_axes(op_kind)
    if pit_axis not in axes:
        raise PlanError(f"axis {pit_axis!r} is not on the sparse operand of {op_kind}")
    proj = shape[:2]
    dim = axes.index(pit_axis)
    if op_kind == "reduce_sum" and pit_axis == "l":
        return (1, 1), ROW_MAJOR
    micro = (1, proj[1]) if dim == 0 else (proj[0], 1)
    return micro, ROW_MAJOR if dim == 0 else COL_MAJOR


def _axis_dim(pit_axis: Union[str, int]) -> int:
    if isinstance(pit_axis, int):
        if pit_axis not in (0, 1):
            raise PlanError(f"pit dimension must be 0 or 1, got {pit_axis}")
        return pit_axis
    if pit_axis not in PIT_DIMS:
        raise PlanError(f"unknown permuted axis {pit_axis!r}")
    return PIT_DIMS[pit_axis]


def micro_occupancy(ann: SparsityAnnotation, micro_tile) -> np.ndarray:
    """Live flag per grid-anchored micro-tile from block-grid prefix sums."""
    t = (int(micro_tile[0]), int(micro_tile[1]))
    cnt = ann.bits().astype(np.int64)
    for axis in (0, 1):
        ext, g = ann.tensor_shape[axis], ann.granularity[axis]
        n = -(-ext // t[axis])
        i = np.arange(n)
        lo = (i * t[axis]) // g
        hi = -(-np.minimum((i + 1) * t[axis], ext) // g)
        pre = np.concatenate([np.zeros((1,) + cnt.shape[1:] if axis == 0 else (cnt.shape[0], 1), np.int64),
                              np.cumsum(cnt, axis=axis)], axis=axis)
        cnt = np.take(pre, hi, axis=axis) - np.take(pre, lo, axis=axis)
    return cnt > 0


def cover_group_counts(ann: SparsityAnnotation, micro_tile, pit_axis: Union[str, int]) -> np.ndarray:
    return micro_occupancy(ann, micro_tile).sum(axis=_axis_dim(pit_axis), dtype=np.int64)


def cover_count(ann: SparsityAnnotation, micro_tile, pit_axis: Union[str, int] = 0) -> int:
    _axis_dim(pit_axis)
    return int(micro_occupancy(ann, micro_tile).sum())


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


def dense_launches(plan: SparseKernelPlan) -> int:
    ext = plan.extents
    if plan.op_kind == "matmul":
        m, k, n = plan.tile.tile_shape
        return _cdiv(ext["m"], m) * _cdiv(ext["k"], k) * _cdiv(ext["n"], n)
    p, l = plan.tile.tile_shape
    return _cdiv(ext["p"], p) * _cdiv(ext["l"], l)


def launches_from_counts(plan: SparseKernelPlan, counts: np.ndarray) -> int:
    """Logical launches for per-group live counts (executor accounting, executor.py:375-423)."""
    if plan.op_kind == "matmul":
        m, k, n = plan.tile.tile_shape
        chunk = m if plan.pit_axis == "m" else k
        return int(np.sum(-(-np.asarray(counts, np.int64) // chunk))) * _cdiv(plan.extents["n"], n)
    p, l = plan.tile.tile_shape
    if plan.pit_axis == "p":
        return int(np.sum(-(-np.asarray(counts, np.int64) // p)))
    return _cdiv(int(np.sum(-(-np.asarray(counts, np.int64) // l))), p)


def plan_launches(plan: SparseKernelPlan, ann: Optional[SparsityAnnotation]) -> int:
    if plan.is_dense:
        return dense_launches(plan)
    assert ann is not None and plan.micro_tile is not None
    axes = sparse_operand_axes(plan.op_kind)
    dim = axes.index(plan.pit_axis)
    return launches_from_counts(plan, cover_group_counts(ann, plan.micro_tile, dim))


def estimate_plan_cost(plan: SparseKernelPlan, ann: Optional[SparsityAnnotation]) -> float:
    if not plan.is_dense and ann is not None:
        want = sparse_operand_shape(plan.op_kind, plan.extents)
        if tuple(ann.tensor_shape) != want:
            raise PlanError(f"annotation shape {ann.tensor_shape} does not match operand {want}")
    return plan_launches(plan, ann) * plan.tile_cost


def forced_plan(
    expr: TensorExpr,
    pit_axis: str,
    registry: KernelRegistry,
    profile=None,
    tile_shape: Optional[Sequence[int]] = None,
) -> SparseKernelPlan:
    op_kind = operator_kind(expr)
    if op_kind not in DEFAULT_TILES:
        raise PlanError(f"cannot execute op kind {op_kind!r}")
    shape = tuple(tile_shape) if tile_shape is not None else DEFAULT_TILES[op_kind]
    tile = registry.get(op_kind, shape)
    if tile is None:
        raise PlanError(f"no registered {op_kind} tile {shape}")
    cost = profile.cost(tile) if profile is not None else 0.0
    extents = {s: expr.extent(s) for s in expr.symbols()}
    if pit_axis == DENSE:
        return SparseKernelPlan(op_kind, DENSE, None, tile, cost, 0.0, ROW_MAJOR, extents)
    micro, layout = get_micro_tile(op_kind, shape, pit_axis)
    return SparseKernelPlan(op_kind, pit_axis, micro, tile, cost, 0.0, layout, extents)


def format_plan(plan: SparseKernelPlan) -> str:
    micro = "-" if plan.micro_tile is None else "x".join(map(str, plan.micro_tile))
    return (
        f"plan op={plan.op_kind} pit_axis={plan.pit_axis} microtile={micro} "
        f"tile={'x'.join(map(str, plan.tile.tile_shape))} impl={plan.tile.impl_id} cost={plan.estimated_cost:.6e}"
    )


# ------------------------------------------------------------------------- Alg. 1 selection
@dataclass(frozen=True)
class PlanCandidate:
    plan: SparseKernelPlan
    total_micro_tiles: int
    total_launches: int
    total_cost: float


class _SampleCovers:
    """Per-sample live micro-tile counts per group, memoised by (micro-tile, axis): tiles whose
    projections coincide (e.g. every tile with M_t = 32 under pit:k) share one count.

    With a GPU visible the counts for every candidate come from one ``pit_cover_counts`` call per
    sample (the detection kernel's occupancy pass, counts only); otherwise from the host prefix-sum
    restatement. Both are exact integer counts of the same rule."""

    def __init__(self, samples: Sequence[SparsityAnnotation], keys=(), device: Optional[bool] = None):
        self.samples = list(samples)
        self._memo: dict = {}
        if device is None:
            device = _gpu_visible()
        keys = list(dict.fromkeys(keys))
        if device and keys and self.samples:
            from .index import cover_counts_device

            per_sample = [cover_counts_device(a, keys) for a in self.samples]
            for i, key in enumerate(keys):
                self._memo[key] = [counts[i] for counts in per_sample]

    def counts(self, micro, dim: int) -> list:
        key = (tuple(micro), dim)
        if key not in self._memo:
            self._memo[key] = [cover_group_counts(a, micro, dim) for a in self.samples]
        return self._memo[key]


def _gpu_visible() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def _preference(c: PlanCandidate):
    # cheapest; on ties dense first, then the larger tile (fewer launches), then impl id
    return (c.total_cost, not c.plan.is_dense, -c.plan.tile.flops, c.plan.tile.impl_id)


def selection_candidates(expr: TensorExpr, samples, registry: KernelRegistry, profile, allow_dense: bool = True):
    """All (tile, PIT axis) plans and the dense fallbacks, each costed as Σ_samples launches x the
    profiled tile cost, sorted by preference (reference policy.py:201-276 contract, error messages
    included). Dense costs `dense_launches` per sample (one sweep when there are no samples)."""
    from dataclasses import replace

    from .expr import pit_axes

    op_kind = operator_kind(expr)
    if op_kind not in ("matmul", "reduce_sum"):
        raise PlanError(f"selection supports matmul and reduce_sum, got {op_kind}")
    extents = {s: expr.extent(s) for s in expr.symbols()}
    tiles = sorted(registry.by_op(op_kind), key=lambda d: d.impl_id)
    if not tiles:
        raise PlanError(f"registry has no {op_kind} tiles")
    want = sparse_operand_shape(op_kind, extents)
    bad = next((a for a in samples if tuple(a.tensor_shape) != want), None)
    if bad is not None:
        raise PlanError(f"sample shape {bad.tensor_shape} does not match operand {want}")
    axes = [a for a in sparse_operand_axes(op_kind) if a in pit_axes(expr)]
    if not axes and not allow_dense:
        raise PlanError("no applicable permuted axis and dense fallback disabled")
    op_axes = sparse_operand_axes(op_kind)
    keys = [(get_micro_tile(op_kind, t.tile_shape, a)[0], op_axes.index(a)) for t in tiles for a in axes]
    covers = _SampleCovers(samples, keys)
    n_samples = len(samples)
    out = []
    for tile in tiles:
        cost = profile.cost(tile)
        for axis in axes if n_samples else ():
            micro, layout = get_micro_tile(op_kind, tile.tile_shape, axis)
            plan = SparseKernelPlan(op_kind, axis, micro, tile, cost, 0.0, layout, dict(extents))
            per = covers.counts(micro, op_axes.index(axis))
            launches = sum(launches_from_counts(plan, c) for c in per)
            total = launches * cost
            out.append(PlanCandidate(replace(plan, estimated_cost=total / n_samples),
                                     int(sum(int(c.sum()) for c in per)), launches, total))
        if allow_dense:
            plan = SparseKernelPlan(op_kind, DENSE, None, tile, cost, 0.0, ROW_MAJOR, dict(extents))
            sweeps = max(n_samples, 1)
            launches = dense_launches(plan) * sweeps
            total = launches * cost
            out.append(PlanCandidate(replace(plan, estimated_cost=total / sweeps), launches, launches, total))
    if not out:
        raise PlanError("no viable plan candidates")
    out.sort(key=_preference)
    return out


def kernel_selection(expr: TensorExpr, samples, registry: KernelRegistry, profile, allow_dense: bool = True):
    """Alg. 1 (reference policy.py:279-292): the cheapest candidate. Scaling every profiled cost by a
    positive constant cannot change the winner; all-dense samples fall to the dense tiling via the
    tie-break."""
    return selection_candidates(expr, samples, registry, profile, allow_dense)[0].plan
