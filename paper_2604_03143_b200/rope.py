"""Rotary re-encoding on the device (reference: roundkv/toymodel.py:60-96).

``rope_apply`` / ``rope_recover`` keep the reference's signatures, shape
validation and the zero-delta exact-copy rule.  Host numpy input returns a
host numpy result (computed on the GPU); a CUDA tensor returns a CUDA
tensor.  Angles are formed in float64 exactly as the reference does
(``delta * base^(-2j/D)``), cos/sin are taken in float64 on the device, and
float32 rows are rotated in float64 with one final rounding.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _kernels
from ._device import default_device, is_host, to_device, to_host
from .core import PositionSpan


def _check_rows(k) -> None:
    if len(k.shape) != 3:
        raise ValueError("expected (tokens, heads, head_dim)")
    if k.shape[-1] % 2 != 0:
        raise ValueError("head_dim must be even")


def rope_apply(k, positions, base: float = 10000.0):
    """Rotate each interleaved pair (2j, 2j+1) of ``k`` (T, H, D) by
    ``positions[t] * base^(-2j/D)``; positions may be signed deltas."""
    _check_rows(k)
    pos = np.asarray(positions.cpu() if isinstance(positions, torch.Tensor) else positions)
    if pos.shape != (k.shape[0],):
        raise ValueError("one position per token required")
    host = is_host(k)
    dev = k.device if isinstance(k, torch.Tensor) else default_device()
    kd = to_device(k, dev)
    T, H, D = kd.shape
    out = torch.empty_like(kd)
    if T:
        table = _kernels.rope_table(pos.astype(np.int64), D, base, kd.dtype, dev)
        job = _kernels.rows_job(kd, None, 0, out, None, 0, T, tbl_row=0, tbl_stride=1,
                                rotate=1)   # K-only job
        _kernels.rows(_kernels.rows_jobs([job]), T, table, 1, H, D, _kernels.ROWS_BLOCK,
                      kd.dtype, dev)
    return to_host(out) if host else out


def rope_recover(span: PositionSpan, k, base: float = 10000.0):
    """Re-encode K rows from span.old_positions to span.new_positions.  A
    zero-delta span returns an exact copy."""
    if k.shape[0] != len(span):
        raise ValueError("span length must match token count")
    delta = span.delta
    if not delta.any():
        return k.copy() if is_host(k) else k.clone()
    return rope_apply(k, delta, base)
