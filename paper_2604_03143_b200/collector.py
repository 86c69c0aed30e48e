"""The KV Collector (reference: roundkv/pic.py:192-235, collective.py:152-163).

Once per All-Gather round every shared output block's master K/V is read
once from HBM, its K rows are re-rotated from the master's source positions
to each agent's target positions, and K and V are scattered straight into
each agent's paged-pool slots (kernel K1, ``tdkv_collect``).  The
reference instead rotates into a dense per-agent context (pic.py:234) and
copies it into the pool later (trace.py:148-152); both forms are provided:

* ``KVCollector`` / ``CollectPlan`` -- the B200 path: a device-resident
  master arena, a planned round (descriptors + per-job delta table resident
  in HBM) and one K0 + one K1 launch per round, writing the pool.
* ``align_cached`` -- drop-in for ``pic.align_cached`` (same signature,
  same in-place mutation of ``contexts[i][0]``, same ledger law: one
  ``record_rope_call`` per layer per call).  ``skeleton_values`` is the V
  copy the reference performs in ``_skeleton`` (pic.py:203-204).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _kernels, _lib
from ._device import (default_device, dtype_code, is_host, ptr, stream_handle, to_device,
                      to_host, upload)
from .core import LayeredKv
from .ledger import CostLedger

# smem budget per CTA for the double-buffered K+V master tile (3 CTAs / SM)
_TILE_SMEM = 72 * 1024
_SMS = 148


def pick_tile_rows(row_bytes: int, budget: int = _TILE_SMEM) -> int:
    rows = max(1, budget // (4 * row_bytes))
    p = 1
    while p * 2 <= min(rows, 32):
        p *= 2
    return p


class MasterArena:
    """Device rows of every shared segment master, K and V planes of shape
    (L, total_rows, H, D); segment ``s`` occupies rows
    [seg_row0[s], seg_row0[s] + seg_len[s])."""

    def __init__(self, k: torch.Tensor, v: torch.Tensor, seg_row0: np.ndarray,
                 seg_len: np.ndarray, source_positions: Sequence[np.ndarray]) -> None:
        if k.shape != v.shape or k.dim() != 4 or k.device.type != "cuda":
            raise ValueError("arena planes must be matching (L, rows, H, D) CUDA tensors")
        dtype_code(k.dtype)
        self.k = k
        self.v = v
        self.seg_row0 = np.asarray(seg_row0, np.int64)
        self.seg_len = np.asarray(seg_len, np.int64)
        self.source_positions = [np.asarray(p, np.int64) for p in source_positions]

    @classmethod
    def from_segments(cls, segments: Sequence[LayeredKv], dtype: Optional[torch.dtype] = None,
                      device: Optional[torch.device] = None) -> "MasterArena":
        device = device or default_device()
        if not segments:
            raise ValueError("no segments")
        lens = np.array([s.num_tokens for s in segments], np.int64)
        row0 = np.concatenate([[0], np.cumsum(lens)[:-1]])
        first = segments[0]
        dtype = dtype or (first.k.dtype if isinstance(first.k, torch.Tensor) else torch.float32)
        L, H, D = first.num_layers, first.num_heads, first.head_dim
        k = torch.empty((L, int(lens.sum()), H, D), dtype=dtype, device=device)
        v = torch.empty_like(k)
        for s, r0, n in zip(segments, row0, lens):
            if (s.num_layers, s.num_heads, s.head_dim) != (L, H, D):
                raise ValueError("segment masters must share (L, H, D)")
            k[:, r0:r0 + n] = to_device(s.k, device, dtype)
            v[:, r0:r0 + n] = to_device(s.v, device, dtype)
        return cls(k, v, row0, lens, [s.positions for s in segments])

    @property
    def num_layers(self) -> int:
        return int(self.k.shape[0])

    @property
    def num_segments(self) -> int:
        return int(self.seg_len.size)

    @property
    def layer_stride(self) -> int:
        return int(self.k.shape[1] * self.k.shape[2] * self.k.shape[3])

    @property
    def nbytes(self) -> int:
        return 2 * self.k.numel() * self.k.element_size()


@dataclass
class CollectJob:
    """One (agent, shared segment) hit: the segment-relative token order is the
    master's; ``dst_rows[i]`` is where token i lands (a pool slot, or a row of
    a dense staging plane) and ``delta[i] = target - source`` position
    (pic.py:60-61)."""

    segment: int
    dst_rows: np.ndarray
    delta: np.ndarray


class CollectPlan:
    """A round's collector work, planned once and resident on the device.

    Jobs are grouped by segment (input order kept within a segment); every
    job with a constant delta shares one cos/sin row, otherwise it gets one
    row per token.  Master tiles of ``tile_rows`` rows pair with job chunks
    so a launch has enough independent (layer, tile, chunk) items to fill
    all SMs.
    """

    def __init__(self, arena: MasterArena, jobs: Sequence[CollectJob], rope_base: float,
                 tile_rows: Optional[int] = None, device: Optional[torch.device] = None) -> None:
        self.device = device or arena.k.device
        self.arena_rows = int(arena.k.shape[1])
        self.num_layers = arena.num_layers
        self.num_heads = int(arena.k.shape[2])
        self.head_dim = int(arena.k.shape[3])
        self.kv_dtype = arena.k.dtype
        self.rope_base = float(rope_base)
        self.num_jobs = len(jobs)
        row_elems = self.num_heads * self.head_dim
        row_bytes = row_elems * arena.k.element_size()
        self.tile_rows = tile_rows or pick_tile_rows(row_bytes)

        order = sorted(range(len(jobs)), key=lambda i: jobs[i].segment)
        jrec = np.zeros(len(jobs), dtype=_lib.COLLECT_JOB)
        dst_parts, delta_parts = [], []
        dst_off = 0
        tbl_rows = 0
        rotate = False
        self.rows_written = 0
        seg_jobs = {}
        for slot, ji in enumerate(order):
            job = jobs[ji]
            s = int(job.segment)
            n = int(arena.seg_len[s])
            dst = np.asarray(job.dst_rows, np.int64)
            delta = np.asarray(job.delta, np.int64)
            if dst.shape != (n,) or delta.shape != (n,):
                raise ValueError("job rows/deltas must cover the whole segment")
            const = bool(n == 0 or (delta == delta[0]).all())
            jrec[slot] = (dst_off, int(arena.seg_row0[s]), tbl_rows, 0 if const else 1, 0)
            delta_parts.append(delta[:1] if const else delta)
            tbl_rows += 1 if const else n
            rotate |= bool(delta.any())
            dst_parts.append(dst)
            dst_off += n
            self.rows_written += n
            seg_jobs.setdefault(s, []).append(slot)
        self.rotate = rotate

        # (tile, job-chunk) units
        tiles = []
        for s in sorted(seg_jobs):
            r0, n = int(arena.seg_row0[s]), int(arena.seg_len[s])
            for t0 in range(0, n, self.tile_rows):
                tiles.append((s, r0 + t0, min(self.tile_rows, n - t0)))
        base_items = max(1, self.num_layers * len(tiles))
        want = 4 * _SMS * 3
        max_jobs = max((len(v) for v in seg_jobs.values()), default=1)
        nchunk = min(max_jobs, max(1, math.ceil(want / base_items)))
        units = []
        for s, row0, nrows in tiles:
            slots = seg_jobs[s]
            per = max(1, math.ceil(len(slots) / nchunk))
            for c0 in range(0, len(slots), per):
                units.append((row0, nrows, slots[0] + c0, slots[0] + min(c0 + per, len(slots))))
        self.units_host = np.array(units, dtype=_lib.COLLECT_UNIT)
        self.jobs_host = jrec
        self.dst_rows_host = (np.concatenate(dst_parts) if dst_parts
                              else np.empty(0, np.int64))
        self.deltas_host = (np.concatenate(delta_parts) if delta_parts
                            else np.empty(0, np.int64))
        # device residency
        self.d_units = upload(self.units_host, self.device)
        self.d_jobs = upload(self.jobs_host, self.device)
        self.d_dst_rows = torch.from_numpy(self.dst_rows_host).to(self.device)
        self.d_deltas = torch.from_numpy(self.deltas_host).to(self.device)
        self.table = torch.empty((max(tbl_rows, 1), self.head_dim // 2, 2),
                                 dtype=torch.float64 if self.kv_dtype == torch.float32
                                 else torch.float32, device=self.device)

    @property
    def h2d_bytes(self) -> int:
        return (self.units_host.nbytes + self.jobs_host.nbytes + self.dst_rows_host.nbytes
                + self.deltas_host.nbytes)

    def algorithmic_bytes(self, with_v: bool = True) -> int:
        """Master read once + every job's rows written (M + N*M)."""
        planes = 2 if with_v else 1
        row = self.num_heads * self.head_dim * torch.tensor([], dtype=self.kv_dtype).element_size()
        return planes * row * self.num_layers * (self._master_rows() + self.rows_written)

    def _master_rows(self) -> int:
        # rows of the arena that some job reads (each tile counted once)
        seen = set()
        total = 0
        for u in self.units_host:
            key = (int(u["row0"]), int(u["nrows"]))
            if key not in seen:
                seen.add(key)
                total += key[1]
        return total

    def launch(self, arena: MasterArena, dst_k: torch.Tensor, dst_v: Optional[torch.Tensor],
               dst_layer_stride: int, grid_limit: int = 0) -> int:
        """K0 (this round's cos/sin rows) + K1; returns the kernels launched."""
        if arena.k.dtype != self.kv_dtype or dst_k.dtype != self.kv_dtype:
            raise ValueError("arena, destination and plan dtypes differ")
        if self.num_jobs == 0:
            return 0
        launched = 0
        if self.rotate:
            _kernels.rope_table_from_device(self.d_deltas, self.head_dim, self.rope_base,
                                            self.kv_dtype, self.table)
            launched += 1
        with_v = dst_v is not None
        _lib.call("tdkv_collect", ptr(arena.k), ptr(arena.v) if with_v else 0,
                  arena.layer_stride, ptr(self.d_units), int(self.units_host.size),
                  self.tile_rows, ptr(self.d_jobs), ptr(self.d_dst_rows),
                  ptr(self.table) if self.rotate else 0, int(self.rotate), ptr(dst_k),
                  ptr(dst_v) if with_v else 0, int(dst_layer_stride), self.num_layers,
                  self.num_heads, self.head_dim, dtype_code(self.kv_dtype), int(grid_limit),
                  stream_handle(self.device))
        return launched + 1


class KVCollector:
    """Arena + pool binding: plan rounds and collect them into the pool."""

    def __init__(self, arena: MasterArena, pool, rope_base: float = 10000.0,
                 tile_rows: Optional[int] = None) -> None:
        if (arena.num_layers, arena.k.shape[2], arena.k.shape[3]) != (
                pool.num_layers, pool.num_heads, pool.head_dim):
            raise ValueError("arena and pool geometry differ")
        if arena.k.dtype != pool.dtype:
            raise ValueError("arena and pool dtypes differ")
        self.arena = arena
        self.pool = pool
        self.rope_base = float(rope_base)
        self.tile_rows = tile_rows

    def plan(self, jobs: Sequence[CollectJob]) -> CollectPlan:
        return CollectPlan(self.arena, jobs, self.rope_base, self.tile_rows, self.pool.device)

    def plan_members(self, members, segment_of) -> CollectPlan:
        """Jobs from reference-shaped requests: ``members[i].hits`` (each with
        ``.target_idx`` and ``.delta``) and ``members[i].slot_map``;
        ``segment_of(hit)`` names the hit's arena segment."""
        jobs = []
        for m in members:
            slots = m.slot_map.slots
            for hit in m.hits:
                jobs.append(CollectJob(int(segment_of(hit)), slots[np.asarray(hit.target_idx)],
                                       np.asarray(hit.delta, np.int64)))
        return self.plan(jobs)

    def collect(self, plan: CollectPlan, ledger: Optional[CostLedger] = None,
                grid_limit: int = 0) -> int:
        n = plan.launch(self.arena, self.pool.k, self.pool.v, self.pool.layer_stride,
                        grid_limit)
        if ledger is not None and plan.num_jobs:
            for layer in range(plan.num_layers):
                ledger.record_rope_call(layer)
        return n


# ---------------------------------------------------------------------------
# reference-shaped drop-ins (pic.py:192-235)


def _unique_masters(jobs):
    ids, segs = {}, []
    for _, hit in jobs:
        key = id(hit.kv)
        if key not in ids:
            ids[key] = len(segs)
            segs.append(hit.kv)
    return ids, segs


def align_cached(members, contexts, rope_base: float,
                 ledger: Optional[CostLedger] = None) -> None:
    """Rotate every member's cached K rows to their prompt positions.

    Drop-in for pic.align_cached: all hits of all members are rotated by one
    device pass per call (one ledger rotation per layer), and
    ``contexts[i][0][layer][hit.target_idx]`` receives the rotated rows.
    Contexts may be host numpy planes (rows come back over PCIe) or CUDA
    tensors (written on the device).
    """
    jobs = [(i, hit) for i, prep in enumerate(members) for hit in prep.hits]
    if not jobs:
        return
    num_layers = jobs[0][1].kv.num_layers
    ids, segs = _unique_masters(jobs)
    ctx0 = contexts[jobs[0][0]][0]
    device = ctx0.device if isinstance(ctx0, torch.Tensor) else default_device()
    dtype = ctx0.dtype if isinstance(ctx0, torch.Tensor) else torch.float32
    arena = MasterArena.from_segments(segs, dtype=dtype, device=device)
    cjobs, offs = [], []
    off = 0
    for _, hit in jobs:
        n = len(hit.target_idx)
        cjobs.append(CollectJob(ids[id(hit.kv)], np.arange(off, off + n, dtype=np.int64),
                                np.asarray(hit.delta, np.int64)))
        offs.append(off)
        off += n
    plan = CollectPlan(arena, cjobs, rope_base, device=device)
    L, _, H, D = arena.k.shape
    staged = torch.empty((L, off, H, D), dtype=dtype, device=device)
    plan.launch(arena, staged, None, off * H * D)
    if ledger is not None:
        for layer in range(num_layers):
            ledger.record_rope_call(layer)
    _scatter_back(jobs, offs, staged, contexts, plane=0)


def skeleton_values(members, contexts) -> None:
    """The V half of the collector: ``ctx_v[:, hit.target_idx] = hit.kv.v``
    for every hit (pic.py:203-204), done as one K1 copy pass."""
    jobs = [(i, hit) for i, prep in enumerate(members) for hit in prep.hits]
    if not jobs:
        return
    ids, segs = _unique_masters(jobs)
    ctx0 = contexts[jobs[0][0]][1]
    device = ctx0.device if isinstance(ctx0, torch.Tensor) else default_device()
    dtype = ctx0.dtype if isinstance(ctx0, torch.Tensor) else torch.float32
    arena = MasterArena.from_segments(segs, dtype=dtype, device=device)
    # V through the K plane of a K-only, rotation-free collect
    varena = MasterArena(arena.v, arena.v, arena.seg_row0, arena.seg_len, arena.source_positions)
    cjobs, offs = [], []
    off = 0
    for _, hit in jobs:
        n = len(hit.target_idx)
        cjobs.append(CollectJob(ids[id(hit.kv)], np.arange(off, off + n, dtype=np.int64),
                                np.zeros(n, np.int64)))
        offs.append(off)
        off += n
    plan = CollectPlan(varena, cjobs, 10000.0, device=device)
    L, _, H, D = arena.v.shape
    staged = torch.empty((L, off, H, D), dtype=dtype, device=device)
    plan.launch(varena, staged, None, off * H * D)
    _scatter_back(jobs, offs, staged, contexts, plane=1)


def _scatter_back(jobs, offs, staged: torch.Tensor, contexts, plane: int) -> None:
    first = contexts[jobs[0][0]][plane]
    if is_host(first):
        host = to_host(staged)
        for (i, hit), off in zip(jobs, offs):
            n = len(hit.target_idx)
            contexts[i][plane][:, np.asarray(hit.target_idx)] = host[:, off:off + n]
        return
    L, R, H, D = staged.shape
    recs = []
    for (i, hit), off in zip(jobs, offs):
        ctx = contexts[i][plane]
        n = len(hit.target_idx)
        src_rows = torch.arange(off, off + n, device=staged.device, dtype=torch.int64)
        dst_rows = torch.as_tensor(np.asarray(hit.target_idx, np.int64), device=staged.device)
        recs.append((_kernels.rows_job(staged, None, R * H * D, ctx, None,
                                       int(ctx.shape[1]) * H * D, n, src_rows=src_rows,
                                       dst_rows=dst_rows), src_rows, dst_rows))
    arr = _kernels.rows_jobs([r[0] for r in recs])
    _kernels.rows(arr, max(len(h.target_idx) for _, h in jobs), None, L, H, D,
                  _kernels.ROWS_BLOCK, staged.dtype, staged.device)
