"""Device plumbing: tensors, streams, descriptor uploads.

PyTorch is used only for device memory, streams and H2D/D2H copies; every
byte of KV arithmetic runs in libtdkv.so.
"""
from __future__ import annotations

import ctypes
import os
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


def upload_many(arrays, device: Optional[torch.device] = None):
    """Several host arrays in ONE pinned upload (16-byte aligned); returns the
    device byte buffer and one uint8 view of it per array (views share the
    buffer's lifetime)."""
    offs, total = [], 0
    for a in arrays:
        offs.append(total)
        total += (a.nbytes + 15) // 16 * 16
    buf = np.zeros(max(total, 16), np.uint8)
    for a, o in zip(arrays, offs):
        buf[o:o + a.nbytes] = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    d = h2d(buf, device)
    return d, [d[o:o + a.nbytes] for a, o in zip(arrays, offs)]


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


# host threads for the host side of PCIe transfers (numpy's large copies
# release the GIL); TDKV_HOST_THREADS=1 keeps that work on the caller thread
HOST_THREADS = int(os.environ.get("TDKV_HOST_THREADS", min(8, os.cpu_count() or 1)))
_host_pool = None


def host_executor():
    global _host_pool
    if _host_pool is None:
        from concurrent.futures import ThreadPoolExecutor
        _host_pool = ThreadPoolExecutor(HOST_THREADS, thread_name_prefix="tdkv-host")
    return _host_pool


# host bytes go to the device through a ring of two pinned staging buffers
# per device (grown to the largest image seen): the host threads fill one
# buffer in chunks of _STAGE_CHUNK while the previous image's H2D drains from
# the other.  Measured on the B200 box for a 51 MB image: a fresh pinned
# block per call 3.2 ms, H2D chunk by chunk during the fill 2.5 ms, a reused
# buffer filled by 8 threads + one H2D ~1.8 ms (scripts/stage_probe.py).
_STAGE_CHUNK = 2 << 20
_stage_rings: dict = {}
_stage_lock = None
_pinned_inflight: list = []       # (event, source buffer) of direct H2Ds


class _Staging:
    __slots__ = ("buf", "event")

    def __init__(self):
        self.buf = None
        self.event = None


def bytes_to_device(buf, device: torch.device, pad: int = 0):
    """Host bytes (any buffer) -> a device uint8 tensor of len(buf) + pad
    bytes through pinned staging (one H2D on the current stream; large
    images are copied into the staging buffer by the host threads).
    Returns the device tensor; the trailing ``pad`` bytes are unspecified."""
    global _stage_lock
    import threading
    if _stage_lock is None:
        _stage_lock = threading.Lock()
    src = np.frombuffer(buf, np.uint8)
    n = src.size
    out = torch.empty(n + pad, dtype=torch.uint8, device=device)
    lib = _lib.load()
    addr = src.ctypes.data if n else 0
    if n and lib.tdkv_host_is_pinned(addr) and lib.tdkv_host_is_pinned(addr + n - 1):
        # already page-locked (e.g. serialize_many(copy=False) views): one
        # H2D straight from the caller's buffer, kept alive until it drains
        _lib.call("tdkv_copy_h2d", ptr(out), addr, n, stream_handle(device))
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(device))
        with _stage_lock:
            _pinned_inflight[:] = [(e, b) for e, b in _pinned_inflight if not e.query()]
            _pinned_inflight.append((ev, buf))
        return out
    with _stage_lock:
        ring = _stage_rings.setdefault(device, [[_Staging(), _Staging()], 0])
        st = ring[0][ring[1]]
        ring[1] ^= 1
        if st.event is not None:
            st.event.synchronize()          # its previous H2D has drained
        if st.buf is None or st.buf.numel() < n + pad:
            st.buf = torch.empty(max(n + pad, 1 << 20), dtype=torch.uint8, pin_memory=True)
        sv = st.buf.numpy()
        if n < 2 * _STAGE_CHUNK or HOST_THREADS <= 1:
            sv[:n] = src
        else:
            bounds = list(range(0, n, _STAGE_CHUNK)) + [n]

            def fill(c):
                a, b = bounds[c], bounds[c + 1]
                sv[a:b] = src[a:b]

            list(host_executor().map(fill, range(len(bounds) - 1)))
        out.copy_(st.buf[:n + pad], non_blocking=True)
        st.event = torch.cuda.Event()
        st.event.record(torch.cuda.current_stream(device))
    return out


def release_inflight() -> None:
    """Drop the references bytes_to_device keeps to pinned source buffers
    whose H2D has drained (so their pinned blocks can be reused)."""
    if _stage_lock is None:
        return
    with _stage_lock:
        _pinned_inflight[:] = [(e, b) for e, b in _pinned_inflight if not e.query()]
