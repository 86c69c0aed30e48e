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


def tf32_split(x: torch.Tensor, out=None):
    """(hi, lo) tf32 planes of a float32 CUDA tensor (numel % 4 == 0):
    hi = cvt.rna(x), lo = cvt.rna(x - hi), stored as float32 bit patterns."""
    if x.dtype != torch.float32 or not x.is_cuda:
        raise ValueError("tf32_split takes a float32 CUDA tensor")
    x = x if x.is_contiguous() else x.contiguous()
    hi, lo = out if out is not None else (torch.empty_like(x), torch.empty_like(x))
    _lib.call("tdkv_tf32_split", ptr(x), x.numel(), ptr(hi), ptr(lo), stream_handle(x.device))
    return hi, lo


def gemm_tf32x3(a, b, out: torch.Tensor, accumulate: bool = False) -> torch.Tensor:
    """out[m, n] (+)= sum_k a[m, k] * b[n, k] with float32 operands given as
    pre-split (hi, lo) pairs of row-major (M, K) / (N, K) planes (3xTF32 on
    the tensor cores, no split inside the GEMM)."""
    (a_hi, a_lo), (b_hi, b_lo) = a, b
    if a_hi.shape != a_lo.shape or b_hi.shape != b_lo.shape or a_hi.shape[1] != b_hi.shape[1]:
        raise ValueError("expected (hi, lo) planes of a (M, K) and b (N, K)")
    if a_hi.stride() != a_lo.stride() or b_hi.stride() != b_lo.stride():
        raise ValueError("hi and lo planes must share a layout")
    M, K = a_hi.shape
    N = b_hi.shape[0]
    if out.dtype != torch.float32 or out.shape != (M, N) or out.stride(1) != 1:
        raise ValueError("out must be a float32 (M, N) row-major tensor")
    _lib.call("tdkv_gemm_tf32x3", ptr(a_hi), ptr(a_lo), a_hi.stride(0), ptr(b_hi), ptr(b_lo),
              b_hi.stride(0), ptr(out), out.stride(0), M, N, K, int(bool(accumulate)),
              stream_handle(a_hi.device))
    return out
