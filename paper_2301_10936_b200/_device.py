"""Device plumbing: torch for memory and streams, the C ABI for compute.

Every function here either moves bytes (H2D / D2H through pinned staging) or forwards device
pointers to libpit_b200.so; none of them computes a result on the host.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

_NP_TO_CODE = {
    np.dtype(np.float32): _lib.PIT_F32,
    np.dtype(np.float64): _lib.PIT_F64,
    np.dtype(np.float16): _lib.PIT_F16,
    np.dtype(np.uint8): _lib.PIT_U8,
    np.dtype(np.bool_): _lib.PIT_U8,
}
_TORCH_TO_CODE = {
    torch.float32: _lib.PIT_F32,
    torch.float64: _lib.PIT_F64,
    torch.bfloat16: _lib.PIT_BF16,
    torch.float16: _lib.PIT_F16,
    torch.uint8: _lib.PIT_U8,
    torch.bool: _lib.PIT_U8,
}


class DeviceError(RuntimeError):
    pass


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("the PIT hot path runs on a CUDA device (sm_100a); no GPU is visible and there is no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def dtype_code(t) -> int:
    if isinstance(t, torch.Tensor):
        code = _TORCH_TO_CODE.get(t.dtype)
    else:
        code = _NP_TO_CODE.get(np.dtype(t.dtype))
    if code is None:
        raise TypeError(f"unsupported dtype {t.dtype}")
    return code


def to_device(x, *, keep_layout: bool = True) -> torch.Tensor:
    """Host array -> device tensor (pinned staging, non-blocking). Device tensors pass through."""
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        return x if x.is_cuda else _pinned_upload(x, dev)
    arr = np.asarray(x)
    if arr.dtype == np.bool_:
        arr = arr.view(np.uint8)
    if keep_layout and arr.ndim == 2 and arr.flags.f_contiguous and not arr.flags.c_contiguous:
        return to_device(np.ascontiguousarray(arr.T)).t()  # column-major stays column-major
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return _pinned_upload(t, dev)


def _pinned_upload(t: torch.Tensor, dev) -> torch.Tensor:
    if t.numel() * t.element_size() < (1 << 16):
        return t.to(dev)
    # same strides as the source, so a column-major operand arrives column-major at every size
    # (the small-tensor t.to(dev) path above preserves dense strides too)
    dense_t = t.dim() == 2 and t.t().is_contiguous()
    if not (t.is_contiguous() or dense_t):
        t = t.contiguous()
    staged = torch.empty_strided(t.shape, t.stride(), dtype=t.dtype, pin_memory=True)
    staged.copy_(t)
    return staged.to(dev, non_blocking=True)


def to_host(t: torch.Tensor, like_layout: str = "row_major") -> np.ndarray:
    arr = t.detach().cpu()
    if arr.dtype == torch.bfloat16:
        arr = arr.float()
    out = arr.numpy()
    if like_layout == "col_major":
        return np.asfortranarray(out)
    return np.ascontiguousarray(out)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def check(status: int, exc_type=DeviceError) -> None:
    if status != _lib.PIT_OK:
        msg = _lib.last_error()
        if status == _lib.PIT_ERR_CUDA:
            raise DeviceError(msg)
        raise exc_type(msg)
