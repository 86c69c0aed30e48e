"""Check-layer selection and family election (reference: roundkv/pic.py
166-189, 238-281; collective.py:117-149).

``batched_selection`` is the paper's "one batched difference pass"
(PAPER.md:337-340): the fresh check-layer keys of every member's reused
positions are compared with the cached (collector-rotated) keys in one K4
launch, and every member's important set and deviation score come out of a
second launch.  The cached rows can be read straight from the paged pool
(``cached_rows`` = slots at the check layer), so the collector's output is
never copied.  The fresh keys come from the model's probe forward, which is
outside this path.

Host helpers keep the reference's exact integer semantics:
``recompute_budget`` (pic.py:174-177), ``select_master`` (collective.py:
117-121) and ``mirror_hint_positions`` (collective.py:124-149).
"""
from __future__ import annotations

import math
import threading
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._device import default_device, dtype_code, h2d, is_host, ptr, stream_handle, to_device
from .core import union_sorted
from .ledger import CostLedger


def recompute_budget(fraction: float, shared_count: int) -> int:
    """ceil(fraction * shared_count) with the reference's decimal-noise guard."""
    return int(math.ceil(round(fraction * shared_count, 6)))


def _mags_device(fresh: torch.Tensor, cached: torch.Tensor,
                 cached_rows: Optional[torch.Tensor]) -> torch.Tensor:
    n = int(fresh.shape[0])
    row = int(np.prod(fresh.shape[1:]))
    out = torch.empty(n, dtype=torch.float32, device=fresh.device)
    if n:
        _lib.call("tdkv_keydiff", ptr(fresh), ptr(cached), ptr(cached_rows), n, row,
                  dtype_code(fresh.dtype), ptr(out), stream_handle(fresh.device))
    return out


def key_diff(fresh_k, cached_k):
    """Per-position L2 magnitude of the key difference, shape (T,)."""
    if tuple(fresh_k.shape) != tuple(cached_k.shape):
        raise ValueError("key tensors must have identical shapes")
    host = is_host(fresh_k)
    dev = fresh_k.device if isinstance(fresh_k, torch.Tensor) else default_device()
    f = to_device(fresh_k, dev)
    c = to_device(cached_k, dev, f.dtype)
    out = _mags_device(f, c, None)
    return out.cpu().numpy() if host else out


class _SelectPlan:
    """Member offsets and budgets of one round shape, resident on the device
    (uploaded once; rounds of the same shape reuse it)."""

    def __init__(self, counts: Sequence[int], budgets: Sequence[int], device) -> None:
        counts = np.asarray(counts, np.int64)
        self.m = int(counts.size)
        self.off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self.total = int(self.off[-1])
        self.max_count = int(counts.max(initial=0))
        self.d_off = h2d(self.off, device)
        self.d_budget = h2d(np.asarray(budgets, np.int32), device)
        # results packed densely: member m's indices at the prefix of the budgets
        budgets = np.maximum(np.asarray(budgets, np.int64), 0)
        self.out_off = np.concatenate([[0], np.cumsum(budgets)]).astype(np.int64)
        self.d_out_off = h2d(self.out_off[:-1].copy(), device)
        self.packed = int(self.out_off[-1])


_PLANS: Dict[tuple, _SelectPlan] = {}


def _plan(counts: Sequence[int], device, budgets: Optional[Sequence[int]] = None,
          fraction: Optional[float] = None) -> _SelectPlan:
    """The resident plan of a round shape: budgets given, or ceil(r * n)."""
    counts = counts if type(counts) is tuple else tuple(map(int, counts))
    key = (device.index, counts, tuple(map(int, budgets)) if budgets is not None
           else ("r", float(fraction)))
    p = _PLANS.get(key)
    if p is None:
        if budgets is None:
            budgets = [recompute_budget(fraction, n) for n in counts]
        if len(_PLANS) >= 64:
            _PLANS.clear()
        p = _PLANS[key] = _SelectPlan(counts, budgets, device)
    return p


def _launch_select(mags: torch.Tensor, p: _SelectPlan):
    """K4's selection launch into ONE int32 buffer [counts | deviation bits |
    packed indices] (a single D2H); returns (result offsets, buffer)."""
    m = p.m
    buf = torch.empty(2 * m + max(p.packed, 1), dtype=torch.int32, device=mags.device)
    if m:
        b = buf.data_ptr()
        _lib.call("tdkv_select_important", mags.data_ptr(), p.d_off.data_ptr(),
                  p.d_budget.data_ptr(), p.d_out_off.data_ptr(), m, p.max_count,
                  b + 8 * m, b, b + 4 * m, stream_handle(mags.device))
    return p.out_off, buf


def _select_device(mags: torch.Tensor, counts: Sequence[int], budgets: Sequence[int]):
    """(result offsets, indices, counts, deviations) views of the result buffer."""
    p = _plan(counts, mags.device, budgets=budgets)
    off, buf = _launch_select(mags, p)
    m = p.m
    return off, buf[2 * m:], buf[:m], buf[m:2 * m].view(torch.float32)


def select_important(magnitudes, budget: int) -> np.ndarray:
    """Top-``budget`` magnitudes (largest first, ties to the lower index,
    zeros never taken), returned as sorted int64 indices."""
    n = int(magnitudes.shape[0])
    if n == 0 or budget <= 0:
        return np.empty(0, dtype=np.int64)
    dev = magnitudes.device if isinstance(magnitudes, torch.Tensor) else default_device()
    mags = to_device(magnitudes, dev, torch.float32)
    _, idx, cnt, _ = _select_device(mags, [n], [budget])
    k = int(cnt[0].item())
    return idx[:k].cpu().numpy().astype(np.int64)


def selection_kernels(fresh: torch.Tensor, cached: torch.Tensor,
                      cached_rows: Optional[torch.Tensor], counts: Sequence[int],
                      fraction: float):
    """The two K4 launches on device tensors, no host synchronization.
    Returns (result offsets, int32 result buffer [counts | deviation bits |
    indices]); member m's indices start at result offset m (the prefix of
    the budgets)."""
    mags = _mags_device(fresh, cached, cached_rows)
    return _launch_select(mags, _plan(counts, fresh.device, fraction=fraction))


def batched_selection(fresh, cached, counts: Sequence[int], fraction: float,
                      cached_rows=None, ledger: Optional[CostLedger] = None
                      ) -> List[Tuple[np.ndarray, float]]:
    """One difference pass over every member's reused rows.

    ``fresh`` (R, H, D): the probe forward's check-layer keys of every member's
    shared positions, members concatenated in order with ``counts[m]`` rows
    each; ``cached``: the matching cached keys -- dense (R, H, D), or a
    (rows, H, D) plane (e.g. ``pool.k[check_layer]``) addressed by
    ``cached_rows`` (R,).  Returns per member (member-relative important
    indices ascending, deviation score); members with no rows get
    (empty, 0.0), like probe_and_select (pic.py:244-246)."""
    dev = fresh.device if isinstance(fresh, torch.Tensor) else default_device()
    f = to_device(fresh, dev)
    c = to_device(cached, dev, f.dtype)
    rows = None if cached_rows is None else to_device(np.asarray(cached_rows, np.int64)
                                                     if not isinstance(cached_rows, torch.Tensor)
                                                     else cached_rows, dev)
    if rows is None and tuple(c.shape) != tuple(f.shape):
        raise ValueError("key tensors must have identical shapes")
    counts = tuple(map(int, counts))
    if sum(counts) != int(f.shape[0]):
        raise ValueError("member counts must cover every fresh row")
    off, buf = selection_kernels(f, c, rows, counts, fraction)
    if ledger is not None:
        ledger.record_selection_pass()
    m = len(counts)
    # results through pinned memory (a pageable D2H runs several times slower)
    staged = _staging(buf.numel())
    staged[:buf.numel()].copy_(buf, non_blocking=True)
    torch.cuda.current_stream(buf.device).synchronize()
    host = staged.numpy()[:buf.numel()]
    cnt_h = host[:m].tolist()
    sums = host[m:2 * m].view(np.float32).tolist()
    idx_h = host[2 * m:].astype(np.int64)        # one widening (and copy) for every member
    starts = off.tolist()
    empty = np.empty(0, dtype=np.int64)
    return [(idx_h[a:a + k], d) if n else (empty.copy(), 0.0)
            for n, a, k, d in zip(counts, starts, cnt_h, sums)]


_STAGE = threading.local()


def _staging(n: int) -> torch.Tensor:
    """A reused pinned int32 staging buffer of at least ``n`` elements, one
    per host thread (the caller synchronizes before reading it, so one buffer
    serves every call of that thread; concurrent groups on other threads
    have their own)."""
    buf = getattr(_STAGE, "buf", None)
    if buf is None or buf.numel() < n:
        buf = _STAGE.buf = torch.empty(max(n, 1 << 16), dtype=torch.int32, pin_memory=True)
    return buf


def select_master(deviation_scores: Dict[int, float]) -> int:
    """Request id with the lowest total deviation; ties to the lowest id."""
    if not deviation_scores:
        raise ValueError("cannot elect a master from an empty group")
    return min(deviation_scores.items(), key=lambda kv: (kv[1], kv[0]))[0]


def mirror_hint_positions(member, master, member_important: np.ndarray,
                          master_important: np.ndarray) -> np.ndarray:
    """Positions where a mirror may differ from its master: fresh on either
    side, different cache entry or offset, or either side's important set."""
    if member.num_tokens != master.num_tokens:
        raise ValueError("hints are only defined for equal-length prompts")
    le, lo = np.asarray(member.label_entry), np.asarray(member.label_offset)
    me, mo = np.asarray(master.label_entry), np.asarray(master.label_offset)
    divergent = (le == -1) | (me == -1) | (le != me) | (lo != mo)
    return union_sorted(np.flatnonzero(divergent), member_important, master_important)
