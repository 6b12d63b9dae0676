"""ctypes binding of libpit_b200.so (the C ABI in include/pit_b200.h).

There is no CPU fallback: if the library is missing or CUDA is unavailable, every device
operation raises. ``load()`` builds the library in-tree on first use when nvcc is present.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libpit_b200.so"
# A/B knob for kernel work: PIT_LIB_PATH points at an alternative build of the same library
# (e.g. an older revision built into build_alt/); the product always ships the in-tree build.
if os.environ.get("PIT_LIB_PATH"):
    _LIB_PATH = Path(os.environ["PIT_LIB_PATH"])
_lock = threading.Lock()
_lib = None

# status codes (pit_status)
PIT_OK = 0
PIT_ERR_ARG = 1
PIT_ERR_SHAPE = 2
PIT_ERR_LAYOUT = 3
PIT_ERR_RANGE = 4
PIT_ERR_CUDA = 5
PIT_ERR_UNSUPPORTED = 6

# dtype codes (pit_dtype)
PIT_F32, PIT_F64, PIT_BF16, PIT_F16, PIT_U8 = 0, 1, 2, 3, 4

# plans (pit_plan)
PIT_PLAN_DENSE, PIT_PLAN_PIT_M, PIT_PLAN_PIT_K = 0, 1, 2

EXPORTS = (
    "pit_last_error",
    "pit_abi_version",
    "pit_kernel_launches",
    "pit_index_geometry",
    "pit_build_index_from_tensor",
    "pit_build_index",
    "pit_cover_counts",
    "pit_index_occupancy",
    "pit_index_union",
    "pit_sread",
    "pit_swrite",
    "pit_spmm",
    "pit_spmm_uses_tensor_cores",
    "pit_spmm_workspace_bytes",
    "pit_dense_reference_f64",
    "pit_grouped_gemm",
    "pit_moe_route",
    "pit_moe_plan",
    "pit_moe_recv_plan",
    "pit_gather_rows",
    "pit_pack_groups",
    "pit_scatter_rows_scaled",
    "pit_copy2d_async",
    "pit_reduce_rows",
    "pit_ep_region_layout",
    "pit_ep_region_alloc",
    "pit_ep_region_free",
    "pit_ep_ipc_handle",
    "pit_ep_ipc_open",
    "pit_ep_ipc_close",
    "pit_ep_error",
    "pit_moe_dispatch",
    "pit_moe_recv_plan_ep",
    "pit_moe_signal",
    "pit_moe_combine",
    "pit_sddmm",
    "pit_sddmm_workspace_bytes",
)


class SpmmArgs(C.Structure):
    """Mirror of ``pit_spmm_args``."""

    _fields_ = [
        ("plan", C.c_int),
        ("dtype", C.c_int),
        ("M", C.c_int64),
        ("N", C.c_int64),
        ("K", C.c_int64),
        ("A", C.c_void_p),
        ("sam", C.c_int64),
        ("sak", C.c_int64),
        ("B", C.c_void_p),
        ("ldb", C.c_int64),
        ("C", C.c_void_p),
        ("ldc", C.c_int64),
        ("t0", C.c_int),
        ("t1", C.c_int),
        ("counts", C.c_void_p),
        ("slots", C.c_void_p),
        ("slot_stride", C.c_int64),
        ("n_groups", C.c_int64),
        ("occ", C.c_void_p),
        ("words_per_group", C.c_int64),
        ("rows", C.c_void_p),
        ("n_rows", C.c_void_p),
        ("n_rows_bound", C.c_int64),
        ("force_simt", C.c_int),
        ("batch", C.c_int64),
        ("b_batch_stride", C.c_int64),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_int64),
    ]


class GroupedGemmArgs(C.Structure):
    """Mirror of ``pit_grouped_gemm_args``."""

    _fields_ = [
        ("dtype", C.c_int),
        ("A", C.c_void_p),
        ("lda", C.c_int64),
        ("rows_a", C.c_int64),
        ("B", C.c_void_p),
        ("ldb", C.c_int64),
        ("C", C.c_void_p),
        ("ldc", C.c_int64),
        ("N", C.c_int64),
        ("K", C.c_int64),
        ("G", C.c_int64),
        ("counts", C.c_void_p),
        ("offsets", C.c_void_p),
        ("tile_offsets", C.c_void_p),
        ("row_src", C.c_void_p),
        ("src_stride", C.c_int64),
        ("row_dst", C.c_void_p),
        ("dst_stride", C.c_int64),
        ("row_scale", C.c_void_p),
        ("act", C.c_int),
        ("max_tiles", C.c_int64),
        ("rows_hint", C.c_int64),
    ]


class SddmmArgs(C.Structure):
    """Mirror of ``pit_sddmm_args``."""

    _fields_ = [
        ("dtype", C.c_int),
        ("A", C.c_void_p),
        ("lda", C.c_int64),
        ("B", C.c_void_p),
        ("ldb", C.c_int64),
        ("C", C.c_void_p),
        ("ldc", C.c_int64),
        ("M", C.c_int64),
        ("N", C.c_int64),
        ("K", C.c_int64),
        ("batch", C.c_int64),
        ("unit_counts", C.c_void_p),
        ("unit_slots", C.c_void_p),
        ("unit_slot_stride", C.c_int64),
        ("n_unit_groups", C.c_int64),
        ("occ", C.c_void_p),
        ("words_per_group", C.c_int64),
        ("g0", C.c_int),
        ("g1", C.c_int),
        ("gate", C.c_void_p),
        ("ldgate", C.c_int64),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_int64),
    ]


class EpArgs(C.Structure):
    """Mirror of ``pit_ep_args``."""

    _fields_ = [
        ("rank", C.c_int),
        ("world", C.c_int),
        ("experts_local", C.c_int64),
        ("capacity", C.c_int64),
        ("row_bytes", C.c_int64),
        ("local", C.c_void_p),
        ("peers", C.c_void_p),
    ]


def _declare(lib) -> None:
    i64, i32, vp = C.c_int64, C.c_int, C.c_void_p
    lib.pit_last_error.restype = C.c_char_p
    lib.pit_last_error.argtypes = []
    lib.pit_abi_version.restype = i32
    lib.pit_kernel_launches.restype = C.c_longlong
    lib.pit_kernel_launches.argtypes = []
    lib.pit_index_geometry.argtypes = [i64, i64, i32, i32, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
    lib.pit_build_index_from_tensor.argtypes = [vp, i32, i64, i64, i64, i64, i32, i32, i32, vp, vp, vp, vp]
    lib.pit_build_index.argtypes = [vp, i64, i64, i32, i32, i32, i32, i32, vp, vp, vp, vp]
    lib.pit_index_occupancy.argtypes = [vp, vp, i64, i64, vp, vp, vp]
    lib.pit_cover_counts.argtypes = [vp, i64, i64, i32, i32, i32, vp, vp, i64, vp, vp]
    lib.pit_index_union.argtypes = [vp, i64, i64, vp, vp, vp, vp]
    lib.pit_sread.argtypes = [vp, i32, i64, i64, i64, i32, vp, i64, i64, i32, i32, i32, i64, vp, i64, i32, vp]
    lib.pit_swrite.argtypes = [vp, vp, i32, i64, i64, i64, i32, i64, i64, i32, i32, i32, i64, vp, i64, i32, vp]
    lib.pit_spmm.argtypes = [C.POINTER(SpmmArgs), vp]
    lib.pit_spmm_uses_tensor_cores.argtypes = [C.POINTER(SpmmArgs)]
    lib.pit_spmm_workspace_bytes.argtypes = [C.POINTER(SpmmArgs)]
    lib.pit_spmm_workspace_bytes.restype = i64
    lib.pit_dense_reference_f64.argtypes = [vp, i64, i64, vp, i64, vp, i64, i64, i64, vp]
    lib.pit_grouped_gemm.argtypes = [C.POINTER(GroupedGemmArgs), vp]
    lib.pit_moe_route.argtypes = [vp, i32, i64, i64, vp, vp, vp, vp, vp, vp]
    lib.pit_moe_plan.argtypes = [vp, i64, vp, i64, vp, vp, vp, i64, vp]
    lib.pit_moe_recv_plan.argtypes = [vp, i64, i64, vp, i64, vp, vp]
    lib.pit_gather_rows.argtypes = [vp, i64, vp, i64, i64, vp, i64, vp]
    lib.pit_pack_groups.argtypes = [vp, i64, vp, i64, vp, vp, i64, i64, i64, vp, i64, vp]
    lib.pit_scatter_rows_scaled.argtypes = [vp, i32, i64, vp, i64, i64, vp, vp, i64, vp]
    lib.pit_copy2d_async.argtypes = [vp, i64, vp, i64, i64, i64, vp]
    lib.pit_reduce_rows.argtypes = [vp, i32, i64, i64, i64, vp, i64, i32, i32, vp, vp]
    ep = C.POINTER(EpArgs)
    lib.pit_ep_region_layout.argtypes = [i64, i64, i64, i64, C.POINTER(i64)]
    lib.pit_ep_region_alloc.argtypes = [i64, C.POINTER(vp)]
    lib.pit_ep_region_free.argtypes = [vp]
    lib.pit_ep_ipc_handle.argtypes = [vp, vp]
    lib.pit_ep_ipc_open.argtypes = [vp, C.POINTER(vp)]
    lib.pit_ep_ipc_close.argtypes = [vp]
    lib.pit_ep_error.argtypes = [vp, C.POINTER(i32)]
    lib.pit_moe_dispatch.argtypes = [ep, vp, i64, i64, vp, vp, vp, vp]
    lib.pit_moe_recv_plan_ep.argtypes = [ep, vp, i64, vp, vp]
    lib.pit_moe_signal.argtypes = [ep, vp]
    lib.pit_moe_combine.argtypes = [ep, i32, i64, vp, vp, vp, vp, i64, vp]
    lib.pit_sddmm.argtypes = [C.POINTER(SddmmArgs), vp]
    lib.pit_sddmm_workspace_bytes.argtypes = [C.POINTER(SddmmArgs)]
    lib.pit_sddmm_workspace_bytes.restype = i64
    for name in EXPORTS:
        if name not in ("pit_last_error", "pit_abi_version", "pit_kernel_launches", "pit_spmm_workspace_bytes",
                        "pit_sddmm_workspace_bytes"):
            getattr(lib, name).restype = i32


def library_path() -> Path:
    return _LIB_PATH


def load(build_if_missing: bool = True):
    """Load (building if needed) the CUDA library. Raises if it cannot be loaded."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not _LIB_PATH.exists() and build_if_missing:
            from . import _build

            _build.build()
        if not _LIB_PATH.exists():
            raise RuntimeError(
                f"{_LIB_PATH} is missing: build it with `python -m paper_2301_10936_b200._build` "
                "(the PIT hot path has no CPU fallback)"
            )
        lib = C.CDLL(str(_LIB_PATH))
        _declare(lib)
        _lib = lib
        return lib


def last_error() -> str:
    return load().pit_last_error().decode(errors="replace")


def kernel_launches() -> int:
    """Kernels launched by libpit_b200.so in this process so far."""
    return int(load().pit_kernel_launches())
