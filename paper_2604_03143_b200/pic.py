"""Per-request and grouped recovery on the B200 (reference: roundkv/pic.py
192-316, collective.py:152-187).

Every numeric stage runs on the device: the private prefix prefill and the
probe/refresh forwards (K5: tcgen05 GEMMs + attention), the V copy and the
batched K rotation (K1, the Collector), the check-layer difference pass and
top-k (K4).  Host code keeps the reference's control flow and integer
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
from ._device import default_device
from ._kernels import move_rows
from .collector import align_cached, skeleton_values
from .core import LayeredKv
from .ledger import CostLedger
from .recompute import ToyModel, _forward, refresh


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


def _skeleton(weights, prep, device: torch.device):
    """Context planes with exact private rows and cached V rows in place
    (pic.py:192-205); K rows of hits are filled by the Collector."""
    m = ToyModel.of(weights, device)
    shape = (m.num_layers, int(np.asarray(prep.tokens).size), m.num_heads, m.head_dim)
    ctx_k = torch.zeros(shape, dtype=torch.float32, device=device)
    ctx_v = torch.zeros_like(ctx_k)
    priv = np.asarray(prep.private_idx, np.int64)
    if priv.size:
        n = priv.size
        out_k = torch.empty((m.num_layers, n, m.num_heads, m.head_dim), dtype=torch.float32,
                            device=device)
        out_v = torch.empty_like(out_k)
        zeros = torch.zeros((m.num_layers, n, m.num_heads, m.head_dim), dtype=torch.float32,
                            device=device)
        toks = np.asarray(prep.tokens, np.int64)[priv]
        _forward(m, toks, np.arange(n, dtype=np.int64), np.arange(n, dtype=np.int64), zeros,
                 zeros, m.num_layers, out_k, out_v)
        move_rows(out_k, ctx_k, dst_rows=priv)
        move_rows(out_v, ctx_v, dst_rows=priv)
    return ctx_k, ctx_v


def probe_and_select(weights, members, contexts, cfg, ledger: Optional[CostLedger] = None):
    """Fresh check-layer keys at reused positions, one batched difference
    pass, per-member important sets and deviation (pic.py:238-281)."""
    L = ToyModel.of(weights, contexts[0][0].device).num_layers
    if cfg.check_layer >= L:
        raise ValueError("check_layer out of range for this model")
    live = [i for i, m in enumerate(members) if m.shared_idx.size]
    if not live:
        return [(np.empty(0, dtype=np.int64), 0.0) for _ in members]
    device = contexts[live[0]][0].device
    model = ToyModel.of(weights, device)
    counts = [int(members[i].shared_idx.size) for i in live]
    R = sum(counts)
    shape = (R, model.num_heads, model.head_dim)
    fresh = torch.empty(shape, dtype=torch.float32, device=device)
    cached = torch.empty_like(fresh)
    off = 0
    for i, n in zip(live, counts):
        prep, (ctx_k, ctx_v) = members[i], contexts[i]
        shared = np.asarray(prep.shared_idx, np.int64)
        fix = np.union1d(shared, prep.structural_idx).astype(np.int64)
        k = torch.empty((cfg.check_layer + 1, fix.size, model.num_heads, model.head_dim),
                        dtype=torch.float32, device=device)
        v = torch.empty_like(k)
        _forward(model, np.asarray(prep.tokens, np.int64), np.asarray(prep.positions, np.int64),
                 fix, ctx_k, ctx_v, cfg.check_layer + 1, k, v)
        # the probe's check-layer rows of the shared positions, and the cached
        # (collector-rotated) rows they are compared with
        move_rows(k[cfg.check_layer], fresh, src_rows=np.searchsorted(fix, shared),
                  dst_rows=np.arange(off, off + n))
        move_rows(ctx_k[cfg.check_layer], cached, src_rows=shared,
                  dst_rows=np.arange(off, off + n))
        off += n
    sel = _select.batched_selection(fresh, cached, counts, cfg.recompute_fraction, ledger=ledger)
    out = [(np.empty(0, dtype=np.int64), 0.0)] * len(members)
    for i, (rel, dev) in zip(live, sel):
        out[i] = (members[i].shared_idx[rel], dev)
    return out


def recover_prepared(weights, prep, cfg, ledger: Optional[CostLedger] = None,
                     device: Optional[torch.device] = None) -> RecoveryResult:
    """Serial recovery of one prepared request (pic.py:303-316)."""
    device = device or default_device()
    context = _skeleton(weights, prep, device)
    skeleton_values([prep], [context])
    align_cached([prep], [context], ToyModel.of(weights, device).rope_base, ledger)
    (important, deviation), = probe_and_select(weights, [prep], [context], cfg, ledger)
    refresh(weights, prep, context, important, ledger)
    num = int(np.union1d(important, prep.structural_idx).size)
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
    contexts = [_skeleton(weights, m, device) for m in members]
    skeleton_values(members, contexts)
    align_cached(members, contexts, model.rope_base, ledger)
    selections = probe_and_select(weights, members, contexts, cfg, ledger)
    results: Dict[int, RecoveryResult] = {}
    scores: Dict[int, float] = {}
    important: Dict[int, np.ndarray] = {}
    for prep, context, (imp, dev) in zip(members, contexts, selections):
        refresh(weights, prep, context, imp, ledger)
        kv = LayeredKv(context[0], context[1], np.asarray(prep.positions, np.int64))
        num = int(np.union1d(imp, prep.structural_idx).size)
        results[prep.request_id] = RecoveryResult(prep.request_id, kv, imp, dev, num)
        scores[prep.request_id] = dev
        important[prep.request_id] = imp
    master_id = _select.select_master(scores)
    master = next(m for m in members if m.request_id == master_id)
    hints = {p.request_id: _select.mirror_hint_positions(p, master, important[p.request_id],
                                                         important[master_id])
             for p in members if p.request_id != master_id}
    return results, ReusePlan(group, scores, master_id, important, hints)
