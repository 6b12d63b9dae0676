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


def register_builtin_kernels(include_b200_tiles: bool = False) -> KernelRegistry:
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


# ------------------------------------------------------------------------ cost table (Alg. 1)
import platform  # noqa: E402
import statistics  # noqa: E402
import warnings  # noqa: E402
from dataclasses import replace  # noqa: E402
from pathlib import Path  # noqa: E402
from typing import Union  # noqa: E402

PROFILE_HEADER = "pit-profile v1"
_N_OPERANDS = {"matmul": 3, "reduce_sum": 2, "vec_add": 3}


class ProfileParseError(ValueError):
    def __init__(self, message: str, line: int):
        super().__init__(f"line {line}: {message}")
        self.line = line


@dataclass(frozen=True)
class ProfileTable:
    """Seconds per logical tile launch, keyed by descriptor (reference tiles.py:151-170)."""

    costs: dict
    fingerprint: str
    reps: int
    foreign: bool = False  # measured on another machine (load_profile warns)

    def cost(self, desc: TileKernelDescriptor) -> float:
        cost = self.costs.get(desc)
        if cost is None:
            raise TileError(f"no profiled cost for {desc}")
        return cost

    def scaled(self, factor: float) -> "ProfileTable":
        return replace(self, costs={d: c * factor for d, c in self.costs.items()})

    def __len__(self) -> int:
        return len(self.costs)


def machine_fingerprint() -> str:
    """Host triple (reference tiles.py:173-174) plus the GPU model, so a table profiled on another
    GPU is flagged foreign."""
    host = f"{platform.machine()}/{platform.system()}/python{platform.python_version()}"
    try:
        import torch

        if torch.cuda.is_available():
            return host + "/" + torch.cuda.get_device_name().replace(" ", "_")
    except Exception:  # pragma: no cover
        pass
    return host


def flop_proportional_profile(registry: KernelRegistry, seconds_per_flop: float = 1e-9) -> ProfileTable:
    """Deterministic stand-in table (cost = FLOPs x constant) for selection tests."""
    return ProfileTable({d: d.flops * seconds_per_flop for d in registry}, "synthetic/flop-proportional", 0)


def _device_timer(run, warmup: int, reps: int, reps_inner: int) -> float:
    """Median seconds per call of `run`, CUDA events on the current stream around `reps_inner` calls."""
    import torch

    for _ in range(warmup):
        run()
    samples = []
    for _ in range(reps):
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record()
        for _ in range(reps_inner):
            run()
        stop.record()
        stop.synchronize()
        samples.append(start.elapsed_time(stop) * 1e-3 / reps_inner)
    return statistics.median(samples)


def profile(registry: KernelRegistry, reps: int = 5, warmup: int = 2, reps_inner: int = 20, dtype="bf16",
            extent: int = 2048) -> ProfileTable:
    """Measure each tile's cost on this B200 (reference tiles.py:187-221 times a numpy call per tile).

    A descriptor no longer names a kernel of its own on B200: it fixes the plan's micro-tile. So a
    matmul tile is costed as the sm_100a pit:k kernel its (M_t, 1) micro-tile selects, run over a
    fully live `extent`^3 operand, divided by that plan's logical launch count; reduce_sum tiles time
    the warp-per-row reduction the same way. vec_add is not on the PIT path and gets a nominal cost.
    """
    if reps < 1:
        raise TileError("reps must be >= 1")
    costs = {}
    descs = list(registry)
    if not descs:
        return ProfileTable(costs, machine_fingerprint(), reps)

    import torch

    from . import _device
    from .executor import DenseTensor, run_sparse_reduce_sum, spmm_device
    from .expr import bind_extents, parse_expr
    from .index import build_index_from_tensor
    from .policy import forced_plan, plan_launches

    dev = _device.require_cuda()
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32, "f64": torch.float64}[
        {"float32": "f32", "float64": "f64"}.get(str(getattr(dtype, "__name__", dtype)), str(dtype))]
    gen = torch.Generator(device=dev).manual_seed(0)
    n = extent
    mm = bind_extents(parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=n, k=n, n=n))
    rs = bind_extents(parse_expr("C[p] += A[p,l]"), dict(p=n, l=n))
    A_cm = torch.randn((n, n), device=dev, generator=gen).to(tdt).t()  # column-major: pit:k layout
    B = torch.randn((n, n), device=dev, generator=gen).to(tdt)
    C = torch.empty((n, n), device=dev, dtype=tdt)
    for desc in descs:
        if desc.op_kind == "matmul":
            plan = forced_plan(mm, "k", registry, tile_shape=desc.tile_shape)
            idx = build_index_from_tensor(A_cm, plan.micro_tile, "k")
            run = lambda: spmm_device(plan, A_cm, B, idx, out=C)  # noqa: E731
            launches = plan_launches(plan, None if plan.is_dense else _full_annotation((n, n)))
        elif desc.op_kind == "reduce_sum":
            plan = forced_plan(rs, "dense", registry, tile_shape=desc.tile_shape)
            At = DenseTensor(B)
            run = lambda: run_sparse_reduce_sum(plan, At, None)  # noqa: E731
            launches = plan_launches(plan, None)
        else:
            costs[desc] = desc.flops * 1e-13
            continue
        cost = _device_timer(run, warmup, reps, reps_inner) / launches
        if cost <= 0.0:
            raise TileError(f"clock returned non-positive cost for {desc}")
        costs[desc] = cost
    return ProfileTable(costs, machine_fingerprint(), reps)


def run_tile(desc: TileKernelDescriptor, inputs, out, scratch=None) -> None:
    """One dense tile on the GPU (reference tiles.py:119-148); see executor.run_tile."""
    from .executor import run_tile as _run

    _run(desc, inputs, out, scratch)


def _full_annotation(shape):
    from .sparsity import random_annotation

    return random_annotation(shape, (1, 1), 0.0, seed=0)


def _entry_text(desc: TileKernelDescriptor, cost: float) -> str:
    return " ".join([desc.op_kind, *(str(d) for d in desc.tile_shape), desc.impl_id, f"{cost:.8e}"])


def save_profile(table: ProfileTable, path: Union[str, Path]) -> None:
    """`pit-profile v1` text: header, fingerprint, reps, then one sorted entry per tile with the cost
    at 9 significant digits, so save -> load -> save is byte-stable."""
    order = sorted(table.costs, key=lambda d: (d.op_kind, d.impl_id))
    body = [PROFILE_HEADER, f"fingerprint {table.fingerprint}", f"reps {table.reps}"]
    body += [_entry_text(d, table.costs[d]) for d in order]
    Path(path).write_text("\n".join(body) + "\n")


def _parse_entry(raw: str, line: int):
    fields = raw.split()
    op = fields[0]
    rank = _RANKS.get(op)
    if rank is None or len(fields) != rank + 3:
        raise ProfileParseError(f"malformed entry {raw!r}", line=line)
    try:
        shape = tuple(map(int, fields[1 : rank + 1]))
        cost = float(fields[rank + 2])
    except ValueError:
        raise ProfileParseError(f"malformed entry {raw!r}", line=line) from None
    return TileKernelDescriptor(op, shape, fields[rank + 1], (ROW_MAJOR,) * _N_OPERANDS[op]), cost


def load_profile(path: Union[str, Path]) -> ProfileTable:
    """Parse `pit-profile v1` (reference tiles.py:232-270 format); errors carry the 1-based line.
    A fingerprint from another machine/GPU warns and sets ``foreign``."""
    text = Path(path).read_text().splitlines()
    if not text or text[0].strip() != PROFILE_HEADER:
        raise ProfileParseError(f"expected header {PROFILE_HEADER!r}", line=1)
    if len(text) < 3 or not text[1].startswith("fingerprint ") or not text[2].startswith("reps "):
        raise ProfileParseError("expected 'fingerprint <s>' then 'reps <n>'", line=2)
    fingerprint = text[1].partition(" ")[2]
    reps_field = text[2].split()
    if len(reps_field) < 2 or not reps_field[1].lstrip("-").isdigit():
        raise ProfileParseError("bad reps line", line=3)
    costs = dict(_parse_entry(raw, no) for no, raw in enumerate(text[3:], start=4) if raw.strip())
    foreign = fingerprint != machine_fingerprint()
    if foreign:
        warnings.warn(f"profile fingerprint {fingerprint!r} is not this machine", stacklevel=2)
    return ProfileTable(costs, fingerprint, int(reps_field[1]), foreign)
