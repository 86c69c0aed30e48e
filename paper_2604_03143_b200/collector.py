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

import ctypes
import math
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _kernels, _lib
from ._device import (HOST_THREADS, default_device, dtype_code, h2d, host_executor, is_host, ptr,
                      stream_handle, to_device, to_host, upload, upload_many)
from .core import LayeredKv
from .ledger import CostLedger

# smem budget per CTA for the double-buffered K+V master tile (3 CTAs / SM)
_TILE_SMEM = int(os.environ.get("TDKV_TILE_SMEM", 32 * 1024))
_SMS = 148
# (layer, tile, job-chunk) work items a plan aims for (job chunks split until
# the launch has this many items); TDKV_PLAN_ITEMS overrides for A/B runs
_TARGET_ITEMS = int(os.environ.get("TDKV_PLAN_ITEMS", 4 * _SMS))


_AUTO_GRAPH = os.environ.get("TDKV_ROUND_GRAPHS", "1") != "0"
# fused K0 (table rows computed inside K1): for rounds up to this many
# algorithmic bytes (C1: 75 MB), where a second launch is a visible share;
# larger rounds keep K0 (recomputing rows per work item would cost more)
_FUSE_TABLE = os.environ.get("TDKV_FUSE_TABLE", "auto")
_FUSE_TABLE_MAX_BYTES = 1 << 30
_ONE_ITEM_MAX_JOBS = int(os.environ.get("TDKV_ONE_ITEM_MAX_JOBS", 8))


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


def _excl_cumsum(a: np.ndarray) -> np.ndarray:
    out = np.zeros_like(a)
    np.cumsum(a[:-1], out=out[1:])
    return out


@dataclass
class HostPlan:
    """Host half of a CollectPlan (pure numpy; what gets uploaded)."""

    units: np.ndarray            # COLLECT_UNIT records
    jobs: np.ndarray             # COLLECT_JOB records (segment-sorted)
    dst_rows: np.ndarray         # int64, job-major
    deltas: np.ndarray           # int64, one per cos/sin table row
    rotate: bool
    rows_written: int
    master_rows: int


def plan_host(seg_row0: np.ndarray, seg_len: np.ndarray, segments: np.ndarray,
              dst_rows: np.ndarray, deltas: np.ndarray, num_layers: int, tile_rows: int,
              target_items: int = _TARGET_ITEMS) -> HostPlan:
    """Vectorized round planning.  ``segments`` (J,) names each job's
    segment; ``dst_rows``/``deltas`` are the jobs' per-token rows and deltas
    concatenated in job order (job j covers seg_len[segments[j]] tokens)."""
    segments = np.asarray(segments, np.int64)
    dst_rows = np.asarray(dst_rows, np.int64)
    deltas = np.asarray(deltas, np.int64)
    J = segments.size
    if J == 0:
        return HostPlan(np.zeros(0, _lib.COLLECT_UNIT), np.zeros(0, _lib.COLLECT_JOB),
                        np.zeros(0, np.int64), np.zeros(0, np.int64), False, 0, 0)
    lens = np.asarray(seg_len, np.int64)[segments]
    total = int(lens.sum())
    if dst_rows.shape != (total,) or deltas.shape != (total,):
        raise ValueError("job rows/deltas must cover the whole segment")
    if (lens <= 0).any():
        raise ValueError("segments must be non-empty")
    order = np.argsort(segments, kind="stable")
    lens_o = lens[order]
    src_off = _excl_cumsum(lens)[order]
    dst_off = _excl_cumsum(lens_o)
    gather = np.repeat(src_off - dst_off, lens_o) + np.arange(total)
    dst_o = dst_rows[gather]
    delta_o = deltas[gather]
    const = np.minimum.reduceat(delta_o, dst_off) == np.maximum.reduceat(delta_o, dst_off)
    tbl_count = np.where(const, 1, lens_o)
    tbl_row = _excl_cumsum(tbl_count)
    keep = np.repeat(~const, lens_o)
    keep[dst_off] = True
    seg_o = segments[order]
    jobs = np.zeros(J, dtype=_lib.COLLECT_JOB)
    jobs["dst_off"] = dst_off
    jobs["seg_row0"] = np.asarray(seg_row0, np.int64)[seg_o]
    jobs["tbl_row"] = tbl_row
    jobs["tbl_stride"] = (~const).astype(np.int32)

    units, master_rows = _build_units(seg_row0, seg_len, seg_o, num_layers, tile_rows,
                                      target_items)
    return HostPlan(units, jobs, dst_o, delta_o[keep], bool(delta_o.any()), total, master_rows)


def _build_units(seg_row0, seg_len, seg_o: np.ndarray, num_layers: int, tile_rows: int,
                 target_items: int):
    """(tile, job-chunk) units over segment-sorted jobs: enough independent
    (layer, tile, chunk) items to fill every SM, without re-reading master
    tiles more than needed."""
    useg, first, njobs = np.unique(seg_o, return_index=True, return_counts=True)
    n_s = np.asarray(seg_len, np.int64)[useg]
    r0_s = np.asarray(seg_row0, np.int64)[useg]
    nt = (n_s + tile_rows - 1) // tile_rows                 # tiles per segment
    tile_seg = np.repeat(np.arange(useg.size), nt)
    tile_i = np.arange(int(nt.sum())) - np.repeat(_excl_cumsum(nt), nt)
    base_items = max(1, num_layers * tile_seg.size)
    nchunk = min(int(njobs.max()), max(1, math.ceil(target_items / base_items)))
    per = np.maximum(1, -(-njobs // nchunk))                # jobs per chunk, per segment
    nc = -(-njobs // per)                                   # chunks per segment
    nc_t = nc[tile_seg]
    unit_tile = np.repeat(np.arange(tile_seg.size), nc_t)
    unit_c = np.arange(int(nc_t.sum())) - np.repeat(_excl_cumsum(nc_t), nc_t)
    us = tile_seg[unit_tile]
    units = np.zeros(unit_tile.size, dtype=_lib.COLLECT_UNIT)
    units["row0"] = r0_s[us] + tile_i[unit_tile] * tile_rows
    units["nrows"] = np.minimum(tile_rows, n_s[us] - tile_i[unit_tile] * tile_rows)
    jb = first[us] + unit_c * per[us]
    units["job_begin"] = jb
    units["job_end"] = np.minimum(jb + per[us], first[us] + njobs[us])
    return units, int(n_s.sum())


def plan_host_offsets(seg_row0: np.ndarray, seg_len: np.ndarray, segments: np.ndarray,
                      dst_off: np.ndarray, job_delta: np.ndarray, num_layers: int,
                      tile_rows: int, target_items: int = _TARGET_ITEMS) -> HostPlan:
    """Planning when every job's destination rows are a contiguous run of a
    device-resident row table (e.g. the agents' slot maps, see SlotArena):
    job j's token i lands at rows[dst_off[j] + i] and rotates by the
    constant ``job_delta[j]``.  Nothing per-token is built or uploaded.

    Runs in C++ (``tdkv_plan_offsets``): jobs stably sorted by segment, the
    (tile, job-chunk) units of ``_build_units``; tests/test_plan.py checks it
    against the numpy restatement record for record."""
    seg_row0 = np.ascontiguousarray(seg_row0, np.int64)
    seg_len = np.ascontiguousarray(seg_len, np.int64)
    segments = np.ascontiguousarray(segments, np.int64)
    J = segments.size
    dst_off = np.ascontiguousarray(dst_off, np.int64)
    job_delta = np.ascontiguousarray(job_delta, np.int64)
    if dst_off.size != J or job_delta.size != J or seg_row0.size != seg_len.size:
        raise ValueError("plan_host_offsets: one dst_off and one delta per job, "
                         "one row0 per segment length")
    jobs = np.zeros(J, dtype=_lib.COLLECT_JOB)
    deltas = np.zeros(J, np.int64)
    info = np.zeros(4, np.int64)
    # units <= tiles + target_items / L (see tdkv_plan.cu's chunking rule)
    cap = int(((seg_len + tile_rows - 1) // tile_rows).sum()) + target_items // max(1, num_layers) + 1
    units = np.zeros(cap, dtype=_lib.COLLECT_UNIT)
    try:
        _lib.call("tdkv_plan_offsets", int(seg_len.size), seg_row0.ctypes.data,
                  seg_len.ctypes.data, J, segments.ctypes.data, dst_off.ctypes.data,
                  job_delta.ctypes.data, int(num_layers), int(tile_rows), int(target_items),
                  jobs.ctypes.data, deltas.ctypes.data, units.ctypes.data, cap, info.ctypes.data)
    except _lib.TdkvError as e:
        raise ValueError(str(e)) from None
    return HostPlan(units[:int(info[0])], jobs, None, deltas, bool(info[1]), int(info[2]),
                    int(info[3]))


def unit_sources(unit_row0: np.ndarray, seg_row0: np.ndarray, seg_len: np.ndarray,
                 seg_source: np.ndarray) -> np.ndarray:
    """uint8 source of each collect unit: the source of the segment whose row
    range [seg_row0[s], seg_row0[s] + seg_len[s]) holds the unit's first row."""
    seg_row0 = np.asarray(seg_row0, np.int64)
    seg_len = np.asarray(seg_len, np.int64)
    seg_source = np.asarray(seg_source, np.int64)
    if seg_source.size and (seg_source.min() < 0 or seg_source.max() > 255):
        raise ValueError("segment sources must be in [0, 255]")
    live = np.flatnonzero(seg_len > 0)
    order = live[np.argsort(seg_row0[live], kind="stable")]
    r0 = np.asarray(unit_row0, np.int64)
    pos = np.searchsorted(seg_row0[order], r0, side="right") - 1
    if r0.size and (pos.min() < 0 or np.any(r0 >= seg_row0[order[pos]] + seg_len[order[pos]])):
        raise ValueError("a unit lies outside every segment")
    return seg_source[order[pos]].astype(np.uint8)


class SlotArena:
    """The agents' slot maps concatenated and resident on the device (pool
    state, uploaded once at admission): a collect job then only names its
    agent's base row and the target offset of its segment."""

    def __init__(self, slot_maps, device: torch.device) -> None:
        lens = np.array([len(m) for m in slot_maps], np.int64)
        self.base = _excl_cumsum(lens)
        cat = (np.concatenate([np.asarray(m.slots, np.int64) for m in slot_maps])
               if slot_maps else np.zeros(0, np.int64))
        self.rows = h2d(cat, device)


class CollectPlan:
    """A round's collector work, planned once and resident on the device.

    Jobs are grouped by segment (input order kept within a segment); a job
    with a constant delta gets one cos/sin row, otherwise one per token.
    Master tiles of ``tile_rows`` rows pair with job chunks so a launch has
    enough independent (layer, tile, chunk) items to fill all SMs.
    """

    def __init__(self, arena: MasterArena, jobs: Sequence[CollectJob], rope_base: float,
                 tile_rows: Optional[int] = None, device: Optional[torch.device] = None) -> None:
        segs = np.array([int(j.segment) for j in jobs], np.int64)
        for j in jobs:
            n = int(arena.seg_len[int(j.segment)])
            if np.shape(j.dst_rows) != (n,) or np.shape(j.delta) != (n,):
                raise ValueError("job rows/deltas must cover the whole segment")
        dst = (np.concatenate([np.asarray(j.dst_rows, np.int64) for j in jobs]) if jobs
               else np.zeros(0, np.int64))
        dl = (np.concatenate([np.asarray(j.delta, np.int64) for j in jobs]) if jobs
              else np.zeros(0, np.int64))
        self._setup(arena, segs, dst, dl, rope_base, tile_rows, device)

    @classmethod
    def from_arrays(cls, arena: MasterArena, segments: np.ndarray, dst_rows: np.ndarray,
                    deltas: np.ndarray, rope_base: float, tile_rows: Optional[int] = None,
                    device: Optional[torch.device] = None) -> "CollectPlan":
        """Plan from concatenated per-job arrays (no per-job Python objects)."""
        self = cls.__new__(cls)
        self._setup(arena, segments, dst_rows, deltas, rope_base, tile_rows, device)
        return self

    @classmethod
    def from_offsets(cls, arena: MasterArena, segments: np.ndarray, dst_off: np.ndarray,
                     job_delta: np.ndarray, rows: torch.Tensor, rope_base: float,
                     tile_rows: Optional[int] = None) -> "CollectPlan":
        """Plan against a device-resident row table ``rows`` (SlotArena.rows):
        job j's token i lands at rows[dst_off[j] + i]; one delta per job."""
        self = cls.__new__(cls)
        self._setup(arena, segments, None, None, rope_base, tile_rows, rows.device,
                    offsets=(dst_off, job_delta, rows))
        return self

    def _setup(self, arena, segments, dst_rows, deltas, rope_base, tile_rows, device,
               offsets=None) -> None:
        self.device = device or arena.k.device
        self.num_layers = arena.num_layers
        self.num_heads = int(arena.k.shape[2])
        self.head_dim = int(arena.k.shape[3])
        self.kv_dtype = arena.k.dtype
        self.rope_base = float(rope_base)
        row_bytes = self.num_heads * self.head_dim * arena.k.element_size()
        self.tile_rows = tile_rows or pick_tile_rows(row_bytes)
        if offsets is None:
            host = plan_host(arena.seg_row0, arena.seg_len, segments, dst_rows, deltas,
                             self.num_layers, self.tile_rows)
        else:
            host = plan_host_offsets(arena.seg_row0, arena.seg_len, segments, offsets[0],
                                     offsets[1], self.num_layers, self.tile_rows)
        self.host = host
        self.num_jobs = int(host.jobs.size)
        self.rotate = host.rotate
        self.rows_written = host.rows_written
        self.units_host = host.units
        # device residency
        # device residency: units, jobs, deltas (+ rows) in one pinned upload
        arrays = [host.units, host.jobs, host.deltas]
        if offsets is None:
            arrays.append(np.ascontiguousarray(host.dst_rows, np.int64))
        self._d_buf, views = upload_many(arrays, self.device)
        self.d_units, self.d_jobs = views[0], views[1]
        self.d_deltas = views[2].view(torch.int64)
        self.d_dst_rows = views[3].view(torch.int64) if offsets is None else offsets[2]
        self._fast: dict = {}
        # small rounds are launch-bound: compute the cos/sin rows inside K1
        # (one kernel per round) when every job has one constant delta
        self.fuse_table = bool(
            self.rotate and host.jobs.size and (host.jobs["tbl_stride"] == 0).all()
            and (_FUSE_TABLE == "1" or (_FUSE_TABLE != "0"
                                        and self.algorithmic_bytes() <= _FUSE_TABLE_MAX_BYTES)))
        # rotate-half pairs (KVCollector(rope_style="neox")); the reference's
        # interleaved pairs otherwise
        self.neox = False
        # fused small rounds whose tiles carry few jobs run one item per CTA
        # (measured ahead of the persistent form up to ~8 jobs per tile)
        self.one_item = bool(host.units.size) and int(
            (host.units["job_end"] - host.units["job_begin"]).max()) <= _ONE_ITEM_MAX_JOBS
        self.table = torch.empty((max(host.deltas.size, 1), self.head_dim // 2, 2),
                                 dtype=torch.float64 if self.kv_dtype == torch.float32
                                 else torch.float32, device=self.device)

    @property
    def h2d_bytes(self) -> int:
        h = self.host
        dst = h.dst_rows.nbytes if h.dst_rows is not None else 0
        return h.units.nbytes + h.jobs.nbytes + dst + h.deltas.nbytes

    def algorithmic_bytes(self, with_v: bool = True) -> int:
        """Master read once + every job's rows written (M + N*M)."""
        planes = 2 if with_v else 1
        row = self.num_heads * self.head_dim * torch.tensor([], dtype=self.kv_dtype).element_size()
        return planes * row * self.num_layers * (self.host.master_rows + self.rows_written)

    def launch_table(self) -> int:
        """K0: this round's cos/sin rows."""
        if not (self.rotate and self.num_jobs):
            return 0
        _kernels.rope_table_from_device(self.d_deltas, self.head_dim, self.rope_base,
                                        self.kv_dtype, self.table)
        return 1

    def launch_collect(self, arena: MasterArena, dst_k: torch.Tensor,
                       dst_v: Optional[torch.Tensor], dst_layer_stride: int,
                       layers: Optional[tuple] = None, grid_limit: int = 0) -> int:
        """K1 over all layers or the layer range ``layers = (l0, l1)``."""
        if self.neox:
            raise ValueError("rotate-half (neox) plans run through KVCollector.collect "
                             "(tdkv_collect_round); the chunked and multi-source launches "
                             "rotate interleaved pairs only")
        if arena.k.dtype != self.kv_dtype or dst_k.dtype != self.kv_dtype:
            raise ValueError("arena, destination and plan dtypes differ")
        if self.num_jobs == 0:
            return 0
        l0, l1 = layers if layers is not None else (0, self.num_layers)
        if not 0 <= l0 < l1 <= self.num_layers:
            raise ValueError("layer range out of bounds")
        esz = arena.k.element_size()
        a_off = l0 * arena.layer_stride * esz
        d_off = l0 * int(dst_layer_stride) * esz
        with_v = dst_v is not None
        _lib.call("tdkv_collect", ptr(arena.k) + a_off, ptr(arena.v) + a_off if with_v else 0,
                  arena.layer_stride, ptr(self.d_units), int(self.units_host.size),
                  self.tile_rows, ptr(self.d_jobs), ptr(self.d_dst_rows),
                  ptr(self.table) if self.rotate else 0, int(self.rotate), ptr(dst_k) + d_off,
                  ptr(dst_v) + d_off if with_v else 0, int(dst_layer_stride), l1 - l0,
                  self.num_heads, self.head_dim, dtype_code(self.kv_dtype), int(grid_limit),
                  stream_handle(self.device))
        return 1

    def unit_sources(self, seg_source: np.ndarray, seg_row0: np.ndarray,
                     seg_len: np.ndarray) -> np.ndarray:
        """Source index of every unit (see ``unit_sources``)."""
        return unit_sources(self.units_host["row0"], seg_row0, seg_len, seg_source)

    def launch_collect_sources(self, sources: Sequence[MasterArena], d_unit_src: torch.Tensor,
                               dst_k: torch.Tensor, dst_v: Optional[torch.Tensor],
                               dst_layer_stride: int, grid_limit: int = 0) -> int:
        """K1 over every layer, unit u's tile read from ``sources[unit_src[u]]``
        (arenas of identical layout: the local one or peer GPUs' arenas
        mapped over NVLink); ``d_unit_src`` from ``unit_sources``."""
        if self.neox:
            raise ValueError("rotate-half (neox) plans run through KVCollector.collect "
                             "(tdkv_collect_round); the chunked and multi-source launches "
                             "rotate interleaved pairs only")
        if not sources or any(a.k.shape != sources[0].k.shape or a.k.dtype != self.kv_dtype
                              for a in sources):
            raise ValueError("sources must be arenas of one layout and the plan's dtype")
        if dst_k.dtype != self.kv_dtype:
            raise ValueError("destination and plan dtypes differ")
        if self.num_jobs == 0:
            return 0
        with_v = dst_v is not None
        n = len(sources)
        src_k = (ctypes.c_void_p * n)(*[ptr(a.k) for a in sources])
        src_v = (ctypes.c_void_p * n)(*[ptr(a.v) for a in sources])
        _lib.call("tdkv_collect_sources", src_k, src_v if with_v else None, n, ptr(d_unit_src),
                  sources[0].layer_stride, ptr(self.d_units), int(self.units_host.size),
                  self.tile_rows, ptr(self.d_jobs), ptr(self.d_dst_rows),
                  ptr(self.table) if self.rotate else 0, int(self.rotate), ptr(dst_k),
                  ptr(dst_v) if with_v else 0, int(dst_layer_stride), self.num_layers,
                  self.num_heads, self.head_dim, dtype_code(self.kv_dtype), int(grid_limit),
                  stream_handle(self.device))
        return 1

    def launch(self, arena: MasterArena, dst_k: torch.Tensor, dst_v: Optional[torch.Tensor],
               dst_layer_stride: int, grid_limit: int = 0) -> int:
        """K0 + K1 over every layer in one foreign call (tdkv_collect_round:
        both kernels launched with programmatic dependent launch, so K1's
        launch and first tile loads overlap K0); returns the kernels
        launched.  The argument list is built once per (arena, destination,
        stream) and kept as ctypes values (small rounds are launch-bound: C1
        moves 75 MB in ~12 us of DRAM time)."""
        if self.num_jobs == 0:
            return 0
        stream = stream_handle(self.device)
        key = (arena.k.data_ptr(), arena.v.data_ptr(), dst_k.data_ptr(),
               dst_v.data_ptr() if dst_v is not None else 0, int(dst_layer_stride),
               int(grid_limit), stream.value)
        fast = self._fast.get(key)
        if fast is None:
            if arena.k.dtype != self.kv_dtype or dst_k.dtype != self.kv_dtype:
                raise ValueError("arena, destination and plan dtypes differ")
            lib = _lib.load()
            C = ctypes
            n_tbl = int(self.d_deltas.numel()) if self.rotate else 0
            inv = (_kernels.inv_freq_device(self.device, self.head_dim, self.rope_base)
                   if self.rotate else None)
            with_v = dst_v is not None
            args = (C.c_void_p(ptr(self.d_deltas) if n_tbl else 0), C.c_int64(n_tbl),
                    C.c_void_p(ptr(inv) if n_tbl else 0), C.c_void_p(ptr(self.table)),
                    C.c_void_p(ptr(arena.k)), C.c_void_p(ptr(arena.v) if with_v else 0),
                    C.c_int64(arena.layer_stride), C.c_void_p(ptr(self.d_units)),
                    C.c_int32(int(self.units_host.size)), C.c_int32(self.tile_rows),
                    C.c_void_p(ptr(self.d_jobs)), C.c_void_p(ptr(self.d_dst_rows)),
                    C.c_void_p(ptr(dst_k)), C.c_void_p(ptr(dst_v) if with_v else 0),
                    C.c_int64(int(dst_layer_stride)), C.c_int32(self.num_layers),
                    C.c_int32(self.num_heads), C.c_int32(self.head_dim),
                    C.c_int32(dtype_code(self.kv_dtype)), C.c_int32(int(grid_limit)),
                    C.c_int32((_lib.ROUND_FUSE_TABLE if self.fuse_table else 0)
                              | (_lib.ROUND_NEOX if self.neox else 0)
                              | (_lib.ROUND_ONE_ITEM if self.fuse_table and self.one_item
                                 else 0)), stream)
            if len(self._fast) >= 16:
                self._fast.clear()
            # keep the tensors whose addresses are baked in alive with the entry
            fast = self._fast[key] = (lib.tdkv_collect_round, args,
                                      2 if n_tbl and not self.fuse_table else 1,
                                      (arena.k, arena.v, dst_k, dst_v, inv))
        fn, args, kernels, _ = fast
        if fn(*args):
            _lib.raise_last("tdkv_collect_round")
        return kernels


class KVCollector:
    """Arena + pool binding: plan rounds and collect them into the pool."""

    def __init__(self, arena: MasterArena, pool, rope_base: float = 10000.0,
                 tile_rows: Optional[int] = None, rope_style: str = "interleaved") -> None:
        """``rope_style``: "interleaved" -- the reference's pairs (2j, 2j+1),
        toymodel.py:78-82 -- or "neox" (j, j + D/2; GPT-NeoX / Llama), an
        extension for models laid out that way (same angles, same arithmetic)."""
        if rope_style not in ("interleaved", "neox"):
            raise ValueError(f"rope_style must be 'interleaved' or 'neox', got {rope_style!r}")
        self.rope_style = rope_style
        if (arena.num_layers, arena.k.shape[2], arena.k.shape[3]) != (
                pool.num_layers, pool.num_heads, pool.head_dim):
            raise ValueError("arena and pool geometry differ")
        if arena.k.dtype != pool.dtype:
            raise ValueError("arena and pool dtypes differ")
        self.arena = arena
        self.pool = pool
        self.rope_base = float(rope_base)
        self.tile_rows = tile_rows
        # a plan collected twice in a row is captured as a CUDA graph and
        # replayed from then on (TDKV_ROUND_GRAPHS=0 disables)
        self.auto_graph = _AUTO_GRAPH
        self._last = None            # (plan, grid_limit, stream) of the previous collect
        self._graph = None           # (key, RoundGraph)

    def _styled(self, plan: CollectPlan) -> CollectPlan:
        plan.neox = self.rope_style == "neox"
        return plan

    def plan(self, jobs: Sequence[CollectJob]) -> CollectPlan:
        return self._styled(CollectPlan(self.arena, jobs, self.rope_base, self.tile_rows,
                                        self.pool.device))

    def capture(self, plan: CollectPlan) -> "RoundGraph":
        """The round as a replayable CUDA graph (see RoundGraph)."""
        return RoundGraph(self, plan)

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

    def plan_offsets(self, segments, dst_off, job_delta, slot_arena: "SlotArena") -> CollectPlan:
        return self._styled(CollectPlan.from_offsets(self.arena, segments, dst_off, job_delta,
                                                     slot_arena.rows, self.rope_base,
                                                     self.tile_rows))

    def plan_arrays(self, segments, dst_rows, deltas) -> CollectPlan:
        return self._styled(CollectPlan.from_arrays(self.arena, segments, dst_rows, deltas,
                                                    self.rope_base, self.tile_rows,
                                                    self.pool.device))

    def collect(self, plan: CollectPlan, ledger: Optional[CostLedger] = None,
                grid_limit: int = 0) -> int:
        """Run the round (K0 + K1).  A plan collected again right after itself
        (a replayed round) is captured once as a CUDA graph (RoundGraph) and
        replayed: one graph launch per round instead of the launch path."""
        stream = torch.cuda.current_stream(self.pool.device)
        key = (id(plan), int(grid_limit), stream.cuda_stream)
        g = self._graph
        if g is not None and g[0] == key and g[1].plan is plan:
            n = g[1].replay()
        elif (self.auto_graph and plan.num_jobs and self._last is not None
              and self._last[0] is plan and self._last[1:] == key[1:]
              and not torch.cuda.is_current_stream_capturing()):
            graph = RoundGraph(self, plan, grid_limit)   # runs the round once, then captures
            self._graph = (key, graph)
            n = graph.kernels
        else:
            n = plan.launch(self.arena, self.pool.k, self.pool.v, self.pool.layer_stride,
                            grid_limit)
        self._last = (plan,) + key[1:]
        if ledger is not None and plan.num_jobs:
            for layer in range(plan.num_layers):
                ledger.record_rope_call(layer)
        return n

    def stage_from_host(self, host_k: torch.Tensor, host_v: torch.Tensor, chunks: int = 4,
                        copy_stream: Optional[torch.cuda.Stream] = None) -> list:
        """Start filling the arena from (pinned) host memory, layer chunk by
        layer chunk, on a copy stream; returns [(l0, l1, event)] to pass to
        ``collect_staged``.  Planning can proceed on the host meanwhile."""
        arena = self.arena
        L = arena.num_layers
        cur = torch.cuda.current_stream(self.pool.device)
        copy_stream = copy_stream or torch.cuda.Stream(self.pool.device)
        bounds = [round(i * L / chunks) for i in range(chunks + 1)]
        copy_stream.wait_stream(cur)             # arena reuse after the previous round
        events = []
        with torch.cuda.stream(copy_stream):
            for l0, l1 in zip(bounds[:-1], bounds[1:]):
                if l1 > l0:
                    arena.k[l0:l1].copy_(host_k[l0:l1], non_blocking=True)
                    arena.v[l0:l1].copy_(host_v[l0:l1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy_stream)
                    events.append((l0, l1, ev))
        return events

    def collect_staged(self, plan: CollectPlan, events: list,
                       ledger: Optional[CostLedger] = None) -> int:
        """K0, then K1 per landed layer chunk (the PCIe transfer of the next
        chunk overlaps the HBM-bound collector on the current one)."""
        cur = torch.cuda.current_stream(self.pool.device)
        n = plan.launch_table()
        for l0, l1, ev in events:
            cur.wait_event(ev)
            n += plan.launch_collect(self.arena, self.pool.k, self.pool.v, self.pool.layer_stride,
                                     layers=(l0, l1))
        if ledger is not None and plan.num_jobs:
            for layer in range(plan.num_layers):
                ledger.record_rope_call(layer)
        return n

    def collect_from_host(self, plan: CollectPlan, host_k: torch.Tensor, host_v: torch.Tensor,
                          chunks: int = 4, copy_stream: Optional[torch.cuda.Stream] = None,
                          ledger: Optional[CostLedger] = None) -> int:
        """Collect a round whose master blocks arrive from (pinned) host memory."""
        events = self.stage_from_host(host_k, host_v, chunks, copy_stream)
        return self.collect_staged(plan, events, ledger)


class RoundGraph:
    """A planned round captured once as a CUDA graph (K0 + K1 with every
    pointer and size baked in).  ``replay()`` re-runs the round on the
    current stream -- on whatever the arena holds at that moment -- with one
    graph launch instead of the per-kernel launch path; for small rounds
    (C1: two kernels, 38 us) the launch overhead is a visible share."""

    def __init__(self, collector: "KVCollector", plan: CollectPlan, grid_limit: int = 0) -> None:
        self.collector = collector
        self.plan = plan                 # keeps the descriptor buffers alive
        device = collector.pool.device
        pool = collector.pool

        def run():
            return plan.launch(collector.arena, pool.k, pool.v, pool.layer_stride, grid_limit)

        side = torch.cuda.Stream(device)
        side.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(side):    # first launches outside capture (attributes set)
            run()
        torch.cuda.current_stream(device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.kernels = run()
        _lib.note_launches(-self.kernels)     # captured, not run: counted at each replay

    def replay(self) -> int:
        """Run the captured round; returns the kernels it launches (they are
        added to tdkv's launch counter)."""
        self.graph.replay()
        _lib.note_launches(self.kernels)
        return self.kernels


class RoundPipeline:
    """Steady-state rounds whose masters arrive from host memory: two arenas
    alternate, so round r+1's masters stream over PCIe (copy stream) while
    round r is collected from the other arena (compute stream)."""

    def __init__(self, arena: MasterArena, pool, rope_base: float = 10000.0,
                 chunks: int = 7) -> None:
        twin = MasterArena(torch.empty_like(arena.k), torch.empty_like(arena.v), arena.seg_row0,
                           arena.seg_len, arena.source_positions)
        self.collectors = [KVCollector(arena, pool, rope_base), KVCollector(twin, pool, rope_base)]
        self.chunks = chunks
        self.copy_stream = torch.cuda.Stream(pool.device)
        self._pending = None          # (collector index, staged chunk events)
        self._round = 0

    def prime(self, host_k: torch.Tensor, host_v: torch.Tensor) -> None:
        """Start streaming the first round's masters."""
        c = self.collectors[self._round % 2]
        self._pending = (self._round % 2,
                         c.stage_from_host(host_k, host_v, self.chunks, self.copy_stream))

    def step(self, plan: CollectPlan, next_host_k: Optional[torch.Tensor],
             next_host_v: Optional[torch.Tensor], ledger: Optional[CostLedger] = None) -> int:
        """Collect the primed round with ``plan`` (planned against either arena:
        both share the segment table); start streaming the next round's masters
        (if given) into the other arena first, so the transfers overlap."""
        if self._pending is None:
            raise RuntimeError("prime() the pipeline first")
        idx, events = self._pending
        nxt = (idx + 1) % 2
        self._pending = None
        if next_host_k is not None:
            self._pending = (nxt, self.collectors[nxt].stage_from_host(
                next_host_k, next_host_v, self.chunks, self.copy_stream))
        self._round += 1
        return self.collectors[idx].collect_staged(plan, events, ledger)


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


def collect_into_contexts(members, contexts, rope_base: float,
                          ledger: Optional[CostLedger] = None) -> None:
    """``skeleton_values`` + ``align_cached`` in one pass for CUDA contexts:
    one master arena, one plan, one K0 + K1 launch moving K (rotated) and V,
    one scatter of both planes into the members' contexts.  Same results and
    ledger law (one rotation per layer) as the two reference-shaped calls."""
    jobs = [(i, hit) for i, prep in enumerate(members) for hit in prep.hits]
    if not jobs:
        return
    ctx0 = contexts[jobs[0][0]][0]
    if is_host(ctx0):
        skeleton_values(members, contexts)
        align_cached(members, contexts, rope_base, ledger)
        return
    num_layers = jobs[0][1].kv.num_layers
    ids, segs = _unique_masters(jobs)
    device, dtype = ctx0.device, ctx0.dtype
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
    staged_k = torch.empty((L, off, H, D), dtype=dtype, device=device)
    staged_v = torch.empty_like(staged_k)
    plan.launch(arena, staged_k, staged_v, off * H * D)
    if ledger is not None:
        for layer in range(num_layers):
            ledger.record_rope_call(layer)
    _scatter_back(jobs, offs, staged_k, contexts, plane=0, staged_v=staged_v)


# read-backs below this many bytes stay one chunk on the caller thread
_HOST_CHUNK_MIN = 4 << 20


def _put_rows(ctx_plane, tgt, rows) -> None:
    """``ctx_plane[:, tgt] = rows`` -- a slice copy when the targets are one
    contiguous run (prompt segments are)."""
    n = tgt.size
    if n and int(tgt[-1]) - int(tgt[0]) == n - 1 and (n == 1 or (np.diff(tgt) == 1).all()):
        t0 = int(tgt[0])
        ctx_plane[:, t0:t0 + n] = rows
    else:
        ctx_plane[:, tgt] = rows


def _scatter_back_host(jobs, offs, staged: torch.Tensor, contexts, plane: int) -> None:
    """Staged rows (device) -> host numpy contexts.  The D2H goes through
    pinned memory (a pageable read runs several times slower) in chunks of
    whole hits, each chunk's rows handed to a host thread as soon as its copy
    event fires, so PCIe and the host-side writes into the contexts overlap."""
    L, R = staged.shape[0], staged.shape[1]
    pinned = torch.empty(staged.shape, dtype=staged.dtype, pin_memory=True)
    nbytes = staged.numel() * staged.element_size()
    # chunks end at member boundaries (a member's hits stay on one thread, in
    # order, so overlapping targets keep the serial last-write-wins result);
    # one chunk when the read-back is small or two members share a context
    planes = [id(contexts[i][plane]) for i in {i for i, _ in jobs}]
    bounds = [0]
    if nbytes >= _HOST_CHUNK_MIN and HOST_THREADS > 1 and len(set(planes)) == len(planes):
        want = R / min(2 * HOST_THREADS, len(planes))
        for k in range(1, len(jobs)):
            if jobs[k][0] != jobs[k - 1][0] and offs[k] >= want * len(bounds):
                bounds.append(k)
    bounds.append(len(jobs))
    row_of = list(offs) + [R]
    stream = torch.cuda.current_stream(staged.device)
    events = []
    for c in range(len(bounds) - 1):
        r0, r1 = row_of[bounds[c]], row_of[bounds[c + 1]]
        for layer in range(L):
            pinned[layer, r0:r1].copy_(staged[layer, r0:r1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        events.append(ev)

    def work(c):
        events[c].synchronize()
        r0, r1 = row_of[bounds[c]], row_of[bounds[c + 1]]
        part = pinned[:, r0:r1]
        host = part.float().numpy() if staged.dtype == torch.bfloat16 else part.numpy()
        for k in range(bounds[c], bounds[c + 1]):
            i, hit = jobs[k]
            tgt = np.asarray(hit.target_idx)
            o = offs[k] - r0
            _put_rows(contexts[i][plane], tgt, host[:, o:o + tgt.size])

    if len(events) == 1:
        work(0)
    else:
        list(host_executor().map(work, range(len(events))))


def _scatter_back(jobs, offs, staged: torch.Tensor, contexts, plane: int,
                  staged_v: Optional[torch.Tensor] = None) -> None:
    first = contexts[jobs[0][0]][plane]
    if is_host(first):
        _scatter_back_host(jobs, offs, staged, contexts, plane)
        return
    L, R, H, D = staged.shape
    hd = H * D
    esz = staged.element_size()
    # every hit's target rows in one upload; sources are contiguous runs of
    # the staged plane (an address offset, no source index array)
    targets = [np.asarray(hit.target_idx, np.int64) for _, hit in jobs]
    d_rows = h2d(np.concatenate(targets), staged.device)
    base = ptr(d_rows)
    recs, t_off = [], 0
    for (i, hit), off, tgt in zip(jobs, offs, targets):
        ctx = contexts[i][plane]
        # staged_v given: K to contexts[i][0] and V to contexts[i][1] in one record
        src_v = ptr(staged_v) + esz * hd * off if staged_v is not None else 0
        dst_v = ptr(contexts[i][1]) if staged_v is not None else 0
        recs.append((ptr(staged) + esz * hd * off, src_v, R * hd, 0, 0, 0, 0, 0, ptr(ctx), dst_v,
                     int(ctx.shape[1]) * hd, base + 8 * t_off, tgt.size, 0, 0, 0))
        t_off += tgt.size
    _kernels.rows(_kernels.rows_jobs(recs), max(t.size for t in targets), None, L, H, D,
                  _kernels.ROWS_BLOCK, staged.dtype, staged.device)
