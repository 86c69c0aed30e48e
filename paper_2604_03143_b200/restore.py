"""Restoring mirror caches into the paged pool (reference: roundkv/restore.py).

``fused_restore`` is Algorithm 1 of the paper as one K3 launch over every
(layer, block): the source block is the diff payload when the block changed
and the master's rows otherwise (the overlay precedes rotation,
restore.py:5-8), K is re-encoded from span.old to span.new, and K and V go
straight to the pool slots.  No staging planes and no dense mirror exist on
the device.  The ledger receives the reference's accounting
(restore.py:70-104) so the byte laws of the reference tests still hold.

``dense_restore`` is the baseline (restore.py:107-139): materialize the
mirror (K3, identity rows), then rotate + scatter it (K3).

``fused_restore_many`` restores a batch of mirrors in one K0 + one K3
launch (the round-level form used by the benchmark).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np
import torch

from . import _kernels, _lib
from ._device import dtype_code, h2d, ptr, stream_handle, table_dtype, to_device
from .collector import pick_tile_rows, plan_host, plan_host_offsets
from .core import PositionSpan
from .diffstore import MirrorHandle, decode_dense_into
from .ledger import CostLedger
from .paged_pool import PagedPool, SlotMap

_EVENTS = ("load", "swap", "diff", "rope", "write")


def _check_restore_args(mirror: MirrorHandle, span: PositionSpan, slot_map: SlotMap) -> None:
    if mirror.released:
        raise ValueError("cannot restore from a released mirror handle")
    master = mirror.master.kv
    if not np.array_equal(span.old_positions, master.positions):
        raise ValueError("span must start at the mirror's source positions")
    if len(slot_map) != master.num_tokens:
        raise ValueError("slot map must cover one slot per token")


def _check_geometry(mirror: MirrorHandle, pool: PagedPool, slot_map: SlotMap) -> None:
    """The descriptors K3 builds from raw pointers must describe the pool,
    the master and the diff consistently (numpy raises on any mismatch in
    the reference, restore.py:68-99); checked before every launch."""
    kv = mirror.master.kv
    L, T, H, D = (int(x) for x in kv.k.shape)
    if (L, H, D) != (pool.num_layers, pool.num_heads, pool.head_dim):
        raise ValueError(f"master planes (L={L}, H={H}, D={D}) do not match the pool "
                         f"(L={pool.num_layers}, H={pool.num_heads}, D={pool.head_dim})")
    diff = mirror.diff
    if (diff.num_layers, diff.total_tokens, diff.num_heads, diff.head_dim) != (L, T, H, D):
        raise ValueError("diff does not describe this master")
    pool.check_slots(slot_map)


def _delta_rows(delta: np.ndarray):
    """cos/sin rows for a span: one row if the delta is constant, else one per
    token.  Returns (deltas, stride, rotate)."""
    if delta.size == 0 or not delta.any():
        return np.zeros(1, np.int64), 0, 0
    if (delta == delta[0]).all():
        return delta[:1].copy(), 0, 1
    return delta.copy(), 1, 1


def _master_planes(mirror: MirrorHandle, pool: PagedPool):
    kv = mirror.master.kv
    # device masters are used in place; host masters are uploaded per call
    return to_device(kv.k, pool.device, pool.dtype), to_device(kv.v, pool.device, pool.dtype)


# TDKV_RESTORE_FAMILY: "auto" (default) takes the family-restore form when the
# batch has at least _FAMILY_MIN mirrors per master (measured: C2's 49-mirror
# family 2.74 vs 2.89 ms per restore, C3's 24-mirror family 0.77 vs 0.74 ms),
# "1" whenever mirrors share a master, "0" never
_FAMILY_MODE = os.environ.get("TDKV_RESTORE_FAMILY", "auto")
_FAMILY_K1 = _FAMILY_MODE != "0"
_FAMILY_MIN = 1 if _FAMILY_MODE == "1" else 32
_MAX_MASTERS = 16            # sources of one tdkv_restore_family launch


def _pack_upload(arrays, device: torch.device):
    """Several host arrays in ONE pinned upload (16-byte aligned offsets);
    returns the device buffer (keep it alive) and each array's address."""
    offs, total = [], 0
    for a in arrays:
        offs.append(total)
        total += (a.nbytes + 15) // 16 * 16
    buf = np.zeros(max(total, 16), np.uint8)
    for a, o in zip(arrays, offs):
        buf[o:o + a.nbytes] = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    d = h2d(buf, device)
    base = ptr(d)
    return d, [base + o for o in offs]


def _family_restore(mirrors, spans, pool: PagedPool, slot_maps, rope_base: float,
                    grid_limit: int) -> bool:
    """Every mirror of the batch restored by K1 with a diff overlay
    (tdkv_restore_family): each master tile is staged once and written,
    rotated, to all of its mirrors' slots -- the collector round of a family
    (the masters are the sources, the mirrors the agents).  Returns False
    (nothing launched) when the batch does not fit that form."""
    L, H, D = pool.num_layers, pool.num_heads, pool.head_dim
    esz = 4 if pool.dtype == torch.float32 else 2
    row_bytes = H * D * esz
    bs = mirrors[0].diff.block_size
    tile = pick_tile_rows(row_bytes)
    while tile > 1 and bs % tile:
        tile //= 2
    if row_bytes % 16:
        return False
    T = mirrors[0].master.kv.num_tokens
    masters, src_of, mirror_src = [], {}, []
    for m in mirrors:
        key = id(m.master.kv)                # host masters are uploaded once per family
        if key not in src_of:
            mk, mv = _master_planes(m, pool)
            if m.master.kv.num_tokens != T or ptr(mk) % 16 or ptr(mv) % 16:
                return False
            src_of[key] = len(masters)
            masters.append((mk, mv))
        mirror_src.append(src_of[key])
    if len(masters) >= len(mirrors) or len(mirrors) < _FAMILY_MIN * len(masters):
        return False                         # little sharing: K3 per mirror is as good
    dev = pool.device
    nb = (T + bs - 1) // bs
    keep = []
    for g0 in range(0, len(masters), _MAX_MASTERS):      # <= 16 masters per launch
        srcs = masters[g0:g0 + _MAX_MASTERS]
        members = [i for i, f in enumerate(mirror_src) if g0 <= f < g0 + _MAX_MASTERS]
        n_src = len(srcs)
        seg_row0 = np.arange(n_src, dtype=np.int64) * T
        seg_len = np.full(n_src, T, np.int64)
        segs = np.array([mirror_src[i] - g0 for i in members], np.int64)
        deltas = [np.asarray(spans[i].delta, np.int64) for i in members]
        const = all(d.size == 0 or (d == d[0]).all() for d in deltas)
        arrays = []
        if const:
            # destinations: the mirrors' device-resident slot maps, concatenated
            job_delta = np.array([int(d[0]) if d.size else 0 for d in deltas], np.int64)
            rows_dev = torch.cat([slot_maps[i].device_slots(dev) for i in members])
            keep.append(rows_dev)
            host = plan_host_offsets(seg_row0, seg_len, segs,
                                     np.arange(len(members), dtype=np.int64) * T, job_delta,
                                     L, tile)
            if host.rotate:
                # one cos/sin row per distinct shift (a family restored to one
                # offset: the cached one-row table, no K0 launch)
                uniq, inv = np.unique(host.deltas, return_inverse=True)
                host.jobs["tbl_row"] = inv
                const_table = _kernels.rope_table(uniq, D, rope_base, pool.dtype, dev)
        else:
            host = plan_host(seg_row0, seg_len, segs,
                             np.concatenate([np.asarray(slot_maps[i].slots, np.int64)
                                             for i in members]),
                             np.concatenate(deltas), L, tile)
            arrays.append(host.dst_rows)
        # payload slabs and block maps in the plan's job order (jobs sorted
        # by master, stable)
        ovl = np.zeros(len(members), _lib.COLLECT_OVERLAY)
        for row, j in enumerate(np.argsort(segs, kind="stable")):
            dd = mirrors[members[j]].diff.device_form(dev, pool.dtype)
            keep.append(dd)
            ovl[row] = (ptr(dd.pay_k), ptr(dd.pay_v), ptr(dd.map_k), ptr(dd.map_v))
        # one upload: units, jobs, overlays, table deltas (+ rows)
        buf, addrs = _pack_upload([host.units, host.jobs, ovl, host.deltas] + arrays, dev)
        keep.append(buf)
        d_rows = addrs[4] if not const else ptr(rows_dev)
        table = None
        if host.rotate and const:
            table = const_table
            keep.append(table)
        elif host.rotate:
            n_tbl = int(host.deltas.size)
            table = torch.empty((n_tbl, D // 2, 2), dtype=table_dtype(pool.dtype), device=dev)
            _lib.call("tdkv_rope_table", addrs[3], n_tbl,
                      ptr(_kernels.inv_freq_device(dev, D, rope_base)), D // 2,
                      dtype_code(pool.dtype), ptr(table), stream_handle(dev))
            keep.append(table)
        src_k = (ctypes.c_void_p * n_src)(*[ptr(k) for k, _ in srcs])
        src_v = (ctypes.c_void_p * n_src)(*[ptr(v) for _, v in srcs])
        _lib.call("tdkv_restore_family", src_k, src_v, n_src, T, addrs[0],
                  int(host.units.size), tile, addrs[1], len(members), d_rows, addrs[2],
                  nb, bs, ptr(table), int(host.rotate), ptr(pool.k), ptr(pool.v),
                  pool.layer_stride, L, H, D, dtype_code(pool.dtype), int(grid_limit),
                  stream_handle(dev))
    # the uploads and temporaries are stream-ordered: the caching allocators
    # keep their memory valid for the launches queued above
    del keep
    return True


def fused_restore_many(mirrors: Sequence[MirrorHandle], spans: Sequence[PositionSpan],
                       pool: PagedPool, slot_maps: Sequence[SlotMap], rope_base: float,
                       ledger: Optional[CostLedger] = None, grid_limit: int = 0) -> int:
    """Restore every mirror: mirrors sharing masters (a family) in one
    family-restore launch (K0 + K1 with the diff overlay: each master tile
    read once for all of its mirrors), otherwise one K0 + one K3 launch."""
    if not mirrors:
        return 0
    bs = mirrors[0].diff.block_size
    for mirror, span, smap in zip(mirrors, spans, slot_maps):
        _check_restore_args(mirror, span, smap)
        _check_geometry(mirror, pool, smap)
        if mirror.diff.block_size != bs:
            raise ValueError("batched restores must share a block size")
    if _FAMILY_K1 and len(mirrors) > 1 and _family_restore(mirrors, spans, pool, slot_maps,
                                                            rope_base, grid_limit):
        for mirror, smap in zip(mirrors, slot_maps):
            pool.mark_written(smap)
            if ledger is not None:
                _fused_ledger(mirror, ledger)
        return 2
    recs, deltas, tbl_row, const_row = [], [], 0, {}
    max_t, L, H, D = 0, pool.num_layers, pool.num_heads, pool.head_dim
    # host masters are uploaded once per master and the device planes kept
    # alive until the launch: the descriptors hold raw addresses, and a plane
    # freed inside this loop would be reused by the next master's upload
    planes = {}
    for mirror, span, smap in zip(mirrors, spans, slot_maps):
        kv = mirror.master.kv
        T = kv.num_tokens
        if id(kv) not in planes:
            planes[id(kv)] = (kv, _master_planes(mirror, pool))
        mk, mv = planes[id(kv)][1]
        dd = mirror.diff.device_form(pool.device, pool.dtype)
        rows, stride, rotate = _delta_rows(span.delta)
        if stride == 0:
            # constant shifts share one table row per distinct delta (a family
            # restored to one offset needs a one-row table: cached, no K0 launch)
            row = const_row.get(int(rows[0]))
            if row is None:
                row = const_row[int(rows[0])] = tbl_row
                deltas.append(rows)
                tbl_row += 1
        else:
            row = tbl_row
            deltas.append(rows)
            tbl_row += rows.size
        recs.append(_kernels.rows_job(mk, mv, T * H * D, pool.k, pool.v, pool.layer_stride, T,
                                      dst_rows=smap.device_slots(pool.device), pay_k=dd.pay_k,
                                      pay_v=dd.pay_v, map_k=dd.map_k, map_v=dd.map_v,
                                      tbl_row=row, tbl_stride=stride, rotate=rotate))
        max_t = max(max_t, T)
    table = _kernels.rope_table(np.concatenate(deltas), D, rope_base, pool.dtype, pool.device)
    # jobs of one family share the master planes: order the work so each
    # master tile is fetched from DRAM once for all of them
    shared = len({(r[0], r[1]) for r in recs}) < len(recs)
    _kernels.rows(_kernels.rows_jobs(recs), max_t, table, L, H, D, bs, pool.dtype, pool.device,
                  grid_limit, job_minor=shared)
    for mirror, smap in zip(mirrors, slot_maps):
        pool.mark_written(smap)
        if ledger is not None:
            _fused_ledger(mirror, ledger)
    return 2


def _fused_ledger(mirror: MirrorHandle, ledger: CostLedger) -> None:
    kv = mirror.master.kv
    layer_pair = 2 * kv.dense_nbytes // (2 * kv.num_layers)   # one layer's K+V planes
    ledger.record_temp_buffer(2 * layer_pair)
    for layer in range(kv.num_layers):
        ledger.record_moved(layer_pair + mirror.diff.layers[layer].payload_nbytes)


def fused_restore(mirror: MirrorHandle, span: PositionSpan, pool: PagedPool, slot_map: SlotMap,
                  rope_base: float, ledger: Optional[CostLedger] = None,
                  trace: Optional[list] = None) -> None:
    """Load, patch, re-encode and write each layer without a dense mirror.

    Untraced, all layers go in one K3 launch.  With ``trace`` the restore runs
    as one K3 launch per layer in layer order (each launch performs that
    layer's load, swap (the staging ring), diff overlay, rotation and write,
    restore.py:72-99) and the layer's five events are appended once its
    launch is enqueued -- the trace reflects the launches that ran."""
    _check_restore_args(mirror, span, slot_map)
    if trace is None:
        fused_restore_many([mirror], [span], pool, [slot_map], rope_base, ledger)
        return
    _check_geometry(mirror, pool, slot_map)
    kv = mirror.master.kv
    L, T, H, D = kv.k.shape
    diff = mirror.diff
    bs = diff.block_size
    nb = (T + bs - 1) // bs
    mk, mv = _master_planes(mirror, pool)
    dd = diff.device_form(pool.device, pool.dtype)
    rows, stride, rotate = _delta_rows(span.delta)
    table = _kernels.rope_table(rows, D, rope_base, pool.dtype, pool.device)
    slots = slot_map.device_slots(pool.device)
    for layer in range(L):
        job = _kernels.rows_job(mk[layer], mv[layer], 0, pool.k[layer], pool.v[layer], 0, T,
                                dst_rows=slots, pay_k=dd.pay_k, pay_v=dd.pay_v,
                                map_k=dd.map_k[layer * nb:], map_v=dd.map_v[layer * nb:],
                                tbl_row=0, tbl_stride=stride, rotate=rotate)
        _kernels.rows(_kernels.rows_jobs([job]), T, table, 1, H, D, bs, pool.dtype, pool.device)
        trace.extend((event, layer) for event in _EVENTS)
    pool.mark_written(slot_map)
    if ledger is not None:
        _fused_ledger(mirror, ledger)


def dense_restore(mirror: MirrorHandle, span: PositionSpan, pool: PagedPool, slot_map: SlotMap,
                  rope_base: float, ledger: Optional[CostLedger] = None,
                  trace: Optional[list] = None) -> None:
    """Baseline: materialize the dense mirror, then rotate and write it
    (one K3 launch for the whole cache; with ``trace``, one per layer so the
    rope/write events follow the launches)."""
    _check_restore_args(mirror, span, slot_map)
    _check_geometry(mirror, pool, slot_map)
    kv = mirror.master.kv
    diff = mirror.diff
    mk, mv = _master_planes(mirror, pool)
    dense_k = torch.empty_like(mk)
    dense_v = torch.empty_like(mv)
    decode_dense_into(mk, mv, diff, dense_k, dense_v)
    if trace is not None:
        trace.append(("materialize", -1))
    if ledger is not None:
        ledger.record_dense_mirror()
        ledger.record_temp_buffer(kv.dense_nbytes)
        ledger.record_moved(kv.dense_nbytes + diff.payload_nbytes + 2 * kv.dense_nbytes)
    L, T, H, D = dense_k.shape
    rows, stride, rotate = _delta_rows(span.delta)
    table = _kernels.rope_table(rows, D, rope_base, pool.dtype, pool.device)
    slots = slot_map.device_slots(pool.device)
    if trace is None:
        job = _kernels.rows_job(dense_k, dense_v, T * H * D, pool.k, pool.v, pool.layer_stride,
                                T, dst_rows=slots, tbl_row=0, tbl_stride=stride, rotate=rotate)
        _kernels.rows(_kernels.rows_jobs([job]), T, table, L, H, D, _kernels.ROWS_BLOCK,
                      pool.dtype, pool.device)
    else:
        for layer in range(L):
            job = _kernels.rows_job(dense_k[layer], dense_v[layer], 0, pool.k[layer],
                                    pool.v[layer], 0, T, dst_rows=slots, tbl_row=0,
                                    tbl_stride=stride, rotate=rotate)
            _kernels.rows(_kernels.rows_jobs([job]), T, table, 1, H, D, _kernels.ROWS_BLOCK,
                          pool.dtype, pool.device)
            trace.extend([("rope", layer), ("write", layer)])
    pool.mark_written(slot_map)
