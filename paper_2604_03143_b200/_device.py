"""Device plumbing: tensors, streams, descriptor uploads.

PyTorch is used only for device memory, streams and H2D/D2H copies; every
byte of KV arithmetic runs in libtdkv.so.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Union

import numpy as np
import torch

from . import _lib

ArrayLike = Union[np.ndarray, torch.Tensor]


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise _lib.TdkvUnavailable("no CUDA device visible; the tdkv path has no CPU fallback")


def default_device() -> torch.device:
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(device: Optional[torch.device] = None) -> ctypes.c_void_p:
    """The current CUDA stream of ``device`` as a cudaStream_t (the raw
    accessor skips building a torch.cuda.Stream object: ~10x cheaper, and it
    is on every launch path)."""
    if _raw_stream is not None:
        idx = device.index if isinstance(device, torch.device) and device.index is not None \
            else (device if isinstance(device, int) else torch.cuda.current_device())
        return ctypes.c_void_p(_raw_stream(idx))
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return _lib.TDKV_F32
    if dt == torch.bfloat16:
        return _lib.TDKV_BF16
    raise ValueError(f"kv tensors must be float32 or bfloat16, got {dt}")


def table_dtype(dt: torch.dtype) -> torch.dtype:
    """cos/sin table element: float64 pairs for f32 KV, float32 for bf16."""
    return torch.float64 if dt == torch.float32 else torch.float32


def is_host(x) -> bool:
    return isinstance(x, np.ndarray)


def to_device(x: ArrayLike, device: Optional[torch.device] = None,
              dtype: Optional[torch.dtype] = None) -> torch.Tensor:
    """numpy -> device tensor (copy); device tensor -> itself (contiguous)."""
    device = device or default_device()
    if isinstance(x, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(x))
        if dtype is not None:
            t = t.to(dtype)
        return t.to(device, non_blocking=False)
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"expected numpy array or torch tensor, got {type(x)}")
    if x.device.type != "cuda":
        x = x.to(device)
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    return x if x.is_contiguous() else x.contiguous()


def upload(arr: np.ndarray, device: Optional[torch.device] = None) -> torch.Tensor:
    """Raw bytes of a host array (e.g. a descriptor table) onto the device."""
    return h2d(np.ascontiguousarray(arr).view(np.uint8).reshape(-1), device)


def h2d(arr: np.ndarray, device: Optional[torch.device] = None) -> torch.Tensor:
    """Host array -> device tensor through pinned staging, asynchronous on the
    current stream (the caching host allocator keeps the staging buffer alive
    until the copy has run), so descriptor uploads do not serialize behind
    bulk pageable copies."""
    device = device or default_device()
    src = torch.from_numpy(np.ascontiguousarray(arr))
    # never .to(device) from pageable memory: torch follows that copy with a
    # stream synchronize, which would stall the host behind every queued
    # kernel (and serialize back-to-back rounds)
    return src.pin_memory().to(device, non_blocking=True)


def ptr(t: Optional[torch.Tensor]) -> int:
    return 0 if t is None else int(t.data_ptr())


def to_host(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        t = t.float()
    return t.detach().cpu().numpy()
