"""Dense tile descriptors: the (M, K, N) tiles a plan is expressed in.

On B200 a descriptor no longer names a CPU microkernel: it fixes the plan's micro-tile (the
tile's sparse-operand projection, policy.get_micro_tile) and the logical launch accounting that
``ExecStats`` reports (reference tiles.py:36-116). Execution itself always runs the sm_100a
kernels, which tile the gathered data natively (128x256 tcgen05 tiles). The built-in registry
holds the reference's four matmul tiles plus B200-native ones whose projections are the
tensor-core-friendly micro-tiles (128,1) / (1,64).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator, Optional

ROW_MAJOR = "row_major"
COL_MAJOR = "col_major"

_RANKS = {"matmul": 3, "reduce_sum": 2, "vec_add": 1}


class TileError(ValueError):
    pass


@dataclass(frozen=True)
class TileKernelDescriptor:
    op_kind: str
    tile_shape: tuple[int, ...]
    impl_id: str
    layouts: tuple[str, ...] = ()

    def __post_init__(self):
        if self.op_kind not in _RANKS:
            raise TileError(f"unknown op kind {self.op_kind!r}")
        if any(d <= 0 for d in self.tile_shape):
            raise TileError(f"tile dims must be positive, got {self.tile_shape}")
        if len(self.tile_shape) != _RANKS[self.op_kind]:
            raise TileError(f"{self.op_kind} tile needs {_RANKS[self.op_kind]} dims")

    @property
    def flops(self) -> int:
        if self.op_kind == "matmul":
            m, k, n = self.tile_shape
            return 2 * m * k * n
        if self.op_kind == "reduce_sum":
            return self.tile_shape[0] * self.tile_shape[1]
        return self.tile_shape[0]

    def buffer_shapes(self):
        if self.op_kind == "matmul":
            m, k, n = self.tile_shape
            return ((m, k), (k, n)), (m, n)
        if self.op_kind == "reduce_sum":
            p, l = self.tile_shape
            return ((p, l),), (p,)
        p = self.tile_shape[0]
        return ((p,), (p,)), (p,)

    def __str__(self) -> str:
        return f"{self.op_kind} {'x'.join(map(str, self.tile_shape))} [{self.impl_id}]"


class KernelRegistry:
    def __init__(self):
        self._by_impl: dict[str, TileKernelDescriptor] = {}

    def register(self, desc: TileKernelDescriptor) -> None:
        if desc.impl_id in self._by_impl:
            raise TileError(f"duplicate impl_id {desc.impl_id!r}")
        self._by_impl[desc.impl_id] = desc

    def by_op(self, op_kind: str) -> list[TileKernelDescriptor]:
        return [d for d in self._by_impl.values() if d.op_kind == op_kind]

    def get(self, op_kind: str, tile_shape) -> Optional[TileKernelDescriptor]:
        shape = tuple(tile_shape)
        return next((d for d in self._by_impl.values() if d.op_kind == op_kind and d.tile_shape == shape), None)

    def __iter__(self) -> Iterator[TileKernelDescriptor]:
        return iter(self._by_impl.values())

    def __len__(self) -> int:
        return len(self._by_impl)


REFERENCE_MATMUL_TILES = ((16, 32, 128), (8, 32, 128), (32, 64, 32), (32, 32, 32))
# B200-native tiles: the tcgen05 tile is 128 rows x 256 columns x 64 k; these shapes make the
# plan's micro-tile match what one MMA consumes without waste.
B200_MATMUL_TILES = ((128, 64, 256), (64, 64, 256), (256, 64, 256))


def register_builtin_kernels(include_b200_tiles: bool = True) -> KernelRegistry:
    reg = KernelRegistry()
    mm = (ROW_MAJOR,) * 3
    for m, k, n in REFERENCE_MATMUL_TILES:
        reg.register(TileKernelDescriptor("matmul", (m, k, n), f"mm{m}x{k}x{n}", mm))
    if include_b200_tiles:
        for m, k, n in B200_MATMUL_TILES:
            reg.register(TileKernelDescriptor("matmul", (m, k, n), f"tc{m}x{k}x{n}", mm))
    reg.register(TileKernelDescriptor("reduce_sum", (16, 64), "rs16x64", (ROW_MAJOR, ROW_MAJOR)))
    reg.register(TileKernelDescriptor("vec_add", (256,), "va256", (ROW_MAJOR,) * 3))
    return reg
