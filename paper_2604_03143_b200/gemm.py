"""Tensor-core GEMM (tcgen05) used by the selective recompute (K5)."""
from __future__ import annotations

from typing import Optional

import torch

from . import _lib
from ._device import dtype_code, ptr, stream_handle


def gemm_tn(a: torch.Tensor, b: torch.Tensor, out: Optional[torch.Tensor] = None,
            accumulate: bool = False) -> torch.Tensor:
    """out[m, n] (+)= sum_k a[m, k] * b[n, k] on the tensor cores.

    ``a`` (M, K) and ``b`` (N, K) are row-major float32 (3xTF32) or bfloat16
    CUDA tensors with 16-byte aligned rows; ``out`` is float32 (M, N)."""
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[1]:
        raise ValueError("expected a (M, K) and b (N, K)")
    if a.dtype != b.dtype:
        raise ValueError("a and b must share a dtype")
    a = a if a.stride(1) == 1 else a.contiguous()
    b = b if b.stride(1) == 1 else b.contiguous()
    M, K = a.shape
    N = b.shape[0]
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=a.device)
        accumulate = False
    if out.dtype != torch.float32 or out.shape != (M, N) or out.stride(1) != 1:
        raise ValueError("out must be a float32 (M, N) row-major tensor")
    _lib.call("tdkv_gemm", ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(out), out.stride(0),
              M, N, K, dtype_code(a.dtype), int(bool(accumulate)), stream_handle(a.device))
    return out
