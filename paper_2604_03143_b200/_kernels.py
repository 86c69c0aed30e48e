"""Thin typed wrappers over the tdkv C-ABI entry points.

Each wrapper takes torch device tensors, uploads the small descriptor tables
the kernel needs, and launches on the current CUDA stream.
"""
from __future__ import annotations

from functools import lru_cache
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._device import dtype_code, h2d, ptr, stream_handle, table_dtype, upload

ROWS_BLOCK = 32          # tiling of the row mover when no diff geometry applies


def inv_freq_host(head_dim: int, base: float) -> np.ndarray:
    """base^(-2j/D) in float64, the expression of toymodel.py:74."""
    return float(base) ** (-np.arange(0, head_dim, 2, dtype=np.float64) / head_dim)


@lru_cache(maxsize=64)
def _inv_freq_dev(device_index: int, head_dim: int, base: float) -> torch.Tensor:
    return torch.from_numpy(inv_freq_host(head_dim, base)).to(
        torch.device("cuda", device_index))


def inv_freq_device(device: torch.device, head_dim: int, base: float) -> torch.Tensor:
    """The float64 inverse frequencies, resident on ``device`` (cached)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    return _inv_freq_dev(idx, head_dim, float(base))


_ONE_ROW_TABLES: dict = {}


def rope_table(deltas: np.ndarray, head_dim: int, base: float, kv_dtype: torch.dtype,
               device: torch.device) -> torch.Tensor:
    """K0: (n, D/2, 2) cos/sin rows for the given int64 deltas.  One-row
    tables (a constant span shift, the common restore case) are kept per
    (stream, delta, geometry): a repeated shift costs no upload and no launch."""
    deltas = np.ascontiguousarray(deltas, dtype=np.int64)
    n = int(deltas.size)
    if n == 1:
        key = (device.index, torch.cuda.current_stream(device).cuda_stream, int(deltas[0]),
               head_dim, float(base), kv_dtype)
        hit = _ONE_ROW_TABLES.get(key)
        if hit is None:
            if len(_ONE_ROW_TABLES) >= 512:
                _ONE_ROW_TABLES.clear()
            hit = _ONE_ROW_TABLES[key] = _rope_table(deltas, head_dim, base, kv_dtype, device)
        return hit
    return _rope_table(deltas, head_dim, base, kv_dtype, device)


def _rope_table(deltas: np.ndarray, head_dim: int, base: float, kv_dtype: torch.dtype,
                device: torch.device) -> torch.Tensor:
    n = int(deltas.size)
    tdt = table_dtype(kv_dtype)
    out = torch.empty((max(n, 1), head_dim // 2, 2), dtype=tdt, device=device)
    if n == 0:
        return out
    d_deltas = h2d(deltas, device)
    inv = _inv_freq_dev(device.index, head_dim, float(base))
    _lib.call("tdkv_rope_table", ptr(d_deltas), n, ptr(inv), head_dim // 2,
              dtype_code(kv_dtype), ptr(out), stream_handle(device))
    return out


def rope_table_from_device(d_deltas: torch.Tensor, head_dim: int, base: float,
                           kv_dtype: torch.dtype, out: torch.Tensor) -> torch.Tensor:
    """K0 on an already-resident delta vector (used by planned, replayable rounds)."""
    inv = _inv_freq_dev(d_deltas.device.index, head_dim, float(base))
    n = int(d_deltas.numel())
    if n:
        _lib.call("tdkv_rope_table", ptr(d_deltas), n, ptr(inv), head_dim // 2,
                  dtype_code(kv_dtype), ptr(out), stream_handle(d_deltas.device))
    return out


def rows(jobs: np.ndarray, max_tokens: int, table: Optional[torch.Tensor], num_layers: int,
         num_heads: int, head_dim: int, block_size: int, kv_dtype: torch.dtype,
         device: torch.device, grid_limit: int = 0, job_minor: bool = False) -> None:
    """K3 over a ROWS_JOB descriptor array.  ``job_minor`` orders the work
    (layer, block, tile, job) -- for jobs sharing a master (a family), whose
    tiles are then read from DRAM once and from L2 by the other jobs."""
    if jobs.size == 0 or max_tokens == 0:
        return
    esz = 4 if kv_dtype == torch.float32 else 2
    flags, tile = 0, 0
    if _contiguous(jobs, esz):
        flags = _lib.ROWS_CONTIGUOUS
        tile = min(block_size, tile_rows_for(num_heads * head_dim * esz))
    if job_minor and jobs.size > 1 and _JOB_MINOR:
        flags |= _lib.ROWS_JOB_MINOR
    d_jobs = upload(jobs, device)
    _lib.call("tdkv_rows", ptr(d_jobs), int(jobs.size), int(max_tokens), ptr(table),
              num_layers, num_heads, head_dim, block_size, dtype_code(kv_dtype), flags, tile,
              grid_limit, stream_handle(device))


# TDKV_RESTORE_ORDER=job keeps the job-major order for A/B measurement
_JOB_MINOR = __import__("os").environ.get("TDKV_RESTORE_ORDER", "family") != "job"
_ROWS_SMEM = int(__import__("os").environ.get("TDKV_ROWS_SMEM", 72 * 1024))


def tile_rows_for(row_bytes: int, budget: int = _ROWS_SMEM) -> int:
    """Rows per staged tile: double-buffered K+V within ``budget`` bytes."""
    rows = max(1, budget // (4 * row_bytes))
    p = 1
    while p * 2 <= min(rows, 32):
        p *= 2
    return p


def _contiguous(jobs: np.ndarray, esz: int) -> bool:
    """Every job reads whole contiguous source rows from 16-byte aligned
    planes/payloads (the TMA-staged K3 path)."""
    if (jobs["src_rows"] != 0).any():
        return False
    for f in ("src_k", "src_v", "pay_k", "pay_v", "dst_k", "dst_v"):
        if (jobs[f] % 16 != 0).any():
            return False
    for f in ("src_layer_stride", "dst_layer_stride"):
        if ((jobs[f] * esz) % 16 != 0).any():
            return False
    return True


def rows_job(src_k, src_v, src_layer_stride, dst_k, dst_v, dst_layer_stride, num_tokens, *,
             src_rows=None, dst_rows=None, pay_k=None, pay_v=None, map_k=None, map_v=None,
             tbl_row=0, tbl_stride=0, rotate=0) -> tuple:
    return (ptr(src_k), ptr(src_v), int(src_layer_stride), ptr(src_rows), ptr(pay_k),
            ptr(pay_v), ptr(map_k), ptr(map_v), ptr(dst_k), ptr(dst_v), int(dst_layer_stride),
            ptr(dst_rows), int(num_tokens), int(tbl_row), int(tbl_stride), int(rotate))


def rows_jobs(tuples) -> np.ndarray:
    return np.array(list(tuples), dtype=_lib.ROWS_JOB)


def fill_rows(plane: torch.Tensor, rows_dev: torch.Tensor, value: float) -> None:
    """Write ``value`` into the given rows of every layer of a (L, cap, H, D) plane."""
    L, cap, H, D = plane.shape
    if plane.dtype == torch.float32:
        bits = int(np.array([value], np.float32).view(np.uint32)[0])
    else:
        bits = int(torch.tensor([value], dtype=torch.bfloat16).view(torch.int16).item()) & 0xFFFF
    _lib.call("tdkv_fill_rows", ptr(plane), cap * H * D, L, ptr(rows_dev), int(rows_dev.numel()),
              H * D, dtype_code(plane.dtype), bits, stream_handle(plane.device))
