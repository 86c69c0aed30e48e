"""Per-request and grouped recovery on the B200 (reference: roundkv/pic.py
192-316, collective.py:152-187).

Every numeric stage runs on the device: the private prefix prefill and the
probe/refresh forwards (K5: tcgen05 GEMMs + attention), the V copy and the
batched K rotation (K1, the Collector), the check-layer difference pass and
top-k (K4).  A group's members share every launch: one Collector pass, one
batched forward each for the private prefixes, the probe and the refresh,
one selection pass -- results are bit-identical to serial recovery because
every row's arithmetic is independent of the batch.  Host code keeps the reference's control flow and integer
metadata, so ``recover_prepared`` / ``collective_recover`` are drop-ins that
take the reference's ``PreparedRequest`` / ``ReuseGroup`` objects (or
anything with the same attributes) and return ``RecoveryResult`` /
``ReusePlan``-shaped results whose ``kv`` planes are CUDA tensors.

Ledger laws are the reference's: one rotation per layer and one selection
pass per recovery unit (C02), ``record_recomputed`` per refresh.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Optional

import numpy as np
import torch

from . import select as _select
from . import _kernels
from ._device import default_device, h2d, ptr
from .collector import collect_into_contexts
from .core import LayeredKv, union_sorted
from .ledger import CostLedger
from .recompute import ToyModel, forward_many


@dataclass(frozen=True)
class PicConfig:
    """Selective-recompute knobs (pic.py:36-48): fraction of reused positions
    to refresh and the layer whose key differences rank them."""

    recompute_fraction: float = 0.15
    check_layer: int = 1

    def __post_init__(self) -> None:
        if not 0.0 <= self.recompute_fraction <= 1.0:
            raise ValueError("recompute_fraction must be within [0, 1]")
        if self.check_layer < 0:
            raise ValueError("check_layer must be non-negative")


@dataclass(eq=False)
class ReuseGroup:
    """Two or more prepared requests that recover together (collective.py:40-59)."""

    group_id: int
    members: list

    def __post_init__(self) -> None:
        if len(self.members) < 2:
            raise ValueError("a reuse group needs at least two members")
        ids = [m.request_id for m in self.members]
        if len(set(ids)) != len(ids):
            raise ValueError("group member request ids must be distinct")

    @property
    def member_ids(self) -> list:
        return [m.request_id for m in self.members]

    def __len__(self) -> int:
        return len(self.members)


@dataclass(eq=False)
class RecoveryResult:
    request_id: int
    kv: LayeredKv
    important_positions: np.ndarray
    deviation_score: float
    num_recomputed: int


@dataclass(eq=False)
class ReusePlan:
    group: object
    deviation_scores: Dict[int, float]
    master_id: int
    important: Dict[int, np.ndarray]
    mirror_diff_hints: Dict[int, np.ndarray]


def _index_blob(arrays, device):
    """Upload int64 index arrays in one copy; returns (keep-alive tensor,
    device address of each array)."""
    arrays = [np.asarray(x, np.int64) for x in arrays]
    sizes = np.array([x.size for x in arrays], np.int64)
    off = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    blob = h2d(np.concatenate(arrays) if arrays else np.zeros(1, np.int64), device)
    base = ptr(blob)
    return blob, [base + 8 * int(o) for o in off]


def _job(src_k, src_v, src_stride, dst_k, dst_v, dst_stride, n, src_rows=0, dst_rows=0):
    """A K3 row-mover record from raw device addresses (see _kernels.rows_job)."""
    return (src_k, src_v, int(src_stride), src_rows, 0, 0, 0, 0, dst_k, dst_v, int(dst_stride),
            dst_rows, int(n), 0, 0, 0)


def _move(jobs, max_tokens, layers, model, device) -> None:
    if jobs:
        _kernels.rows(_kernels.rows_jobs(jobs), max_tokens, None, layers, model.num_heads,
                      model.head_dim, _kernels.ROWS_BLOCK, torch.float32, device)


def _skeletons(weights, preps, device: torch.device):
    """Context planes of every request with exact private rows (one batched
    prefill of all private prefixes) and zeros elsewhere (pic.py:192-205);
    cached V and rotated K rows are filled by the Collector afterwards."""
    m = ToyModel.of(weights, device)
    L, H, D = m.num_layers, m.num_heads, m.head_dim
    contexts = []
    for prep in preps:
        shape = (L, int(np.asarray(prep.tokens).size), H, D)
        ctx_k = torch.zeros(shape, dtype=torch.float32, device=device)
        contexts.append((ctx_k, torch.zeros_like(ctx_k)))
    privs = [np.asarray(p.private_idx, np.int64) for p in preps]
    items = [(np.asarray(p.tokens, np.int64)[pv], np.arange(pv.size, dtype=np.int64),
              np.arange(pv.size, dtype=np.int64), None, None) for p, pv in zip(preps, privs)]
    if not any(pv.size for pv in privs):
        return contexts
    out_k, out_v, row0 = forward_many(m, items, L)
    R = int(out_k.shape[1])
    keep, dst = _index_blob(privs, device)
    hd = H * D
    jobs = [_job(ptr(out_k) + 4 * hd * int(r0), ptr(out_v) + 4 * hd * int(r0), R * hd,
                 ptr(ck), ptr(cv), int(ck.shape[1]) * hd, pv.size, dst_rows=d)
            for (ck, cv), pv, r0, d in zip(contexts, privs, row0, dst) if pv.size]
    _move(jobs, max(pv.size for pv in privs), L, m, device)
    del keep
    return contexts


def probe_and_select(weights, members, contexts, cfg, ledger: Optional[CostLedger] = None):
    """Fresh check-layer keys at reused positions (one batched probe forward
    of every member), one batched difference pass, per-member important sets
    and deviation (pic.py:238-281)."""
    L = ToyModel.of(weights, contexts[0][0].device).num_layers
    if cfg.check_layer >= L:
        raise ValueError("check_layer out of range for this model")
    live = [i for i, m in enumerate(members) if m.shared_idx.size]
    if not live:
        return [(np.empty(0, dtype=np.int64), 0.0) for _ in members]
    device = contexts[live[0]][0].device
    model = ToyModel.of(weights, device)
    H, D = model.num_heads, model.head_dim
    hd = H * D
    counts = [int(members[i].shared_idx.size) for i in live]
    R = sum(counts)
    fresh = torch.empty((R, H, D), dtype=torch.float32, device=device)
    cached = torch.empty_like(fresh)
    shared = [np.asarray(members[i].shared_idx, np.int64) for i in live]
    fixes = [union_sorted(sh, members[i].structural_idx)
             for i, sh in zip(live, shared)]
    items = [(np.asarray(members[i].tokens, np.int64), np.asarray(members[i].positions, np.int64),
              fx, contexts[i][0], contexts[i][1]) for i, fx in zip(live, fixes)]
    pk, _, row0 = forward_many(model, items, cfg.check_layer + 1, k_only_last=True)
    # the probe's check-layer rows of the shared positions, and the cached
    # (collector-rotated) rows they are compared with, gathered in one launch
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]])
    idx = [np.searchsorted(fx, sh) for fx, sh in zip(fixes, shared)]
    keep, ptrs = _index_blob(idx + shared, device)
    src_fresh, src_cached = ptrs[:len(live)], ptrs[len(live):]
    P = int(pk.shape[1])
    base_fresh = ptr(pk[cfg.check_layer])
    jobs = []
    for j, i in enumerate(live):
        n, o = counts[j], int(offs[j])
        ctx_k = contexts[i][0]
        jobs.append(_job(base_fresh + 4 * hd * int(row0[j]), 0, P * hd,
                         ptr(fresh) + 4 * hd * o, 0, R * hd, n, src_rows=src_fresh[j]))
        jobs.append(_job(ptr(ctx_k[cfg.check_layer]), 0, int(ctx_k.shape[1]) * hd,
                         ptr(cached) + 4 * hd * o, 0, R * hd, n, src_rows=src_cached[j]))
    _move(jobs, max(counts), 1, model, device)
    del keep
    sel = _select.batched_selection(fresh, cached, counts, cfg.recompute_fraction, ledger=ledger)
    out = [(np.empty(0, dtype=np.int64), 0.0)] * len(members)
    for i, (rel, dev) in zip(live, sel):
        out[i] = (members[i].shared_idx[rel], dev)
    return out


def refresh_many(weights, preps, contexts, importants,
                 ledger: Optional[CostLedger] = None) -> None:
    """refresh (pic.py:284-300) of several members as one batched forward:
    important and structural rows recomputed at all layers and written into
    each member's context."""
    if not preps:
        return
    device = contexts[0][0].device
    m = ToyModel.of(weights, device)
    hd = m.num_heads * m.head_dim
    fixes = [union_sorted(imp, p.structural_idx)
             for p, imp in zip(preps, importants)]
    items = [(np.asarray(p.tokens, np.int64), np.asarray(p.positions, np.int64), fx, ck, cv)
             for p, fx, (ck, cv) in zip(preps, fixes, contexts)]
    out_k, out_v, row0 = forward_many(m, items, m.num_layers)
    R = int(out_k.shape[1])
    keep, dst = _index_blob(fixes, device)
    jobs = [_job(ptr(out_k) + 4 * hd * int(r0), ptr(out_v) + 4 * hd * int(r0), R * hd,
                 ptr(ck), ptr(cv), int(ck.shape[1]) * hd, fx.size, dst_rows=d)
            for (ck, cv), fx, r0, d in zip(contexts, fixes, row0, dst) if fx.size]
    _move(jobs, max(fx.size for fx in fixes), m.num_layers, m, device)
    del keep
    if ledger is not None:
        for fx in fixes:
            if fx.size:
                ledger.record_recomputed(int(fx.size))


def recover_prepared(weights, prep, cfg, ledger: Optional[CostLedger] = None,
                     device: Optional[torch.device] = None) -> RecoveryResult:
    """Serial recovery of one prepared request (pic.py:303-316)."""
    device = device or default_device()
    context, = _skeletons(weights, [prep], device)
    collect_into_contexts([prep], [context], ToyModel.of(weights, device).rope_base, ledger)
    (important, deviation), = probe_and_select(weights, [prep], [context], cfg, ledger)
    refresh_many(weights, [prep], [context], [important], ledger)
    num = int(union_sorted(important, prep.structural_idx).size)
    kv = LayeredKv(context[0], context[1], np.asarray(prep.positions, np.int64))
    return RecoveryResult(prep.request_id, kv, important, deviation, num)


def collective_recover(weights, group, cfg, ledger: Optional[CostLedger] = None,
                       device: Optional[torch.device] = None):
    """Grouped recovery: one Collector pass (rotation) and one selection pass
    for all members, then per-member refresh, master election and mirror
    hints (collective.py:152-187)."""
    device = device or default_device()
    members = group.members
    model = ToyModel.of(weights, device)
    contexts = _skeletons(weights, members, device)
    collect_into_contexts(members, contexts, model.rope_base, ledger)
    selections = probe_and_select(weights, members, contexts, cfg, ledger)
    refresh_many(weights, members, contexts, [imp for imp, _ in selections], ledger)
    results: Dict[int, RecoveryResult] = {}
    scores: Dict[int, float] = {}
    important: Dict[int, np.ndarray] = {}
    for prep, context, (imp, dev) in zip(members, contexts, selections):
        kv = LayeredKv(context[0], context[1], np.asarray(prep.positions, np.int64))
        num = int(union_sorted(imp, prep.structural_idx).size)
        results[prep.request_id] = RecoveryResult(prep.request_id, kv, imp, dev, num)
        scores[prep.request_id] = dev
        important[prep.request_id] = imp
    master_id = _select.select_master(scores)
    master = next(m for m in members if m.request_id == master_id)
    hints = {p.request_id: _select.mirror_hint_positions(p, master, important[p.request_id],
                                                         important[master_id])
             for p in members if p.request_id != master_id}
    return results, ReusePlan(group, scores, master_id, important, hints)
