"""Content-addressed segment cache with LRU eviction, on the native index
(reference: roundkv/segment_index.py).

``SegmentIndex`` keeps the reference's API and behaviour (most recent entry
per digest wins a lookup, lookups refresh recency, byte-budget LRU eviction
that skips pinned entries, ``on_evict`` in eviction order,
``PinnedEntryError`` on explicit removal of a pinned entry) with the digest
map, the recency list and the eviction walk in C++ (``tdkv_segidx_*``);
this wrapper owns the entry objects.  ``lookup_many`` resolves every
segment of a round in one native call.
"""
from __future__ import annotations

import ctypes
import itertools
import threading
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from . import _lib


class EmptySegmentError(ValueError):
    """Raised when an entry (or a stream) would cover zero tokens."""


class PinnedEntryError(RuntimeError):
    """Raised when removal of a pinned entry is attempted explicitly."""


_entry_ids = itertools.count()


@dataclass(eq=False)
class SegmentCacheEntry:
    """One cached segment (segment_index.py:56-83): digest, the positions its
    KV was computed at, a store handle, the context digest, its byte size."""

    digest: bytes
    source_positions: np.ndarray
    kv_ref: object
    context_digest: bytes
    nbytes: int
    entry_id: int = field(default_factory=lambda: next(_entry_ids))

    def __post_init__(self) -> None:
        self.source_positions = np.asarray(self.source_positions, dtype=np.int64)
        if self.source_positions.size == 0:
            raise EmptySegmentError("entry must cover at least one token")
        if self.source_positions.size > 1 and not np.all(np.diff(self.source_positions) > 0):
            raise ValueError("source positions must be strictly increasing")
        if self.nbytes <= 0:
            raise ValueError("entry byte size must be positive")


def _digest16(d: bytes) -> bytes:
    """The native key: token digests are 16 bytes (core.token_digest); other
    lengths are folded to 16 by blake2b so any bytes key still works."""
    if len(d) == 16:
        return d if type(d) is bytes else bytes(d)
    import hashlib
    return hashlib.blake2b(bytes(d), digest_size=16, person=b"tdkv-segidx").digest()


class SegmentIndex:
    """Digest-keyed cache of SegmentCacheEntry with byte-budget LRU eviction
    (segment_index.py:86-183)."""

    def __init__(self, budget_bytes: int,
                 is_pinned: Optional[Callable[[object], bool]] = None,
                 on_evict: Optional[Callable[[SegmentCacheEntry], None]] = None) -> None:
        if budget_bytes < 0:
            raise ValueError("budget must be non-negative")
        self.budget_bytes = int(budget_bytes)
        self._is_pinned = is_pinned or (lambda ref: False)
        self._on_evict = on_evict
        self._lib = _lib.load()
        self._h = self._lib.tdkv_segidx_create(self.budget_bytes)
        if not self._h:
            raise MemoryError("tdkv_segidx_create failed")
        # native ids are assigned here (entries from other code may carry
        # colliding entry_id counters): native id -> entry, entry -> native id
        self._entries: Dict[int, SegmentCacheEntry] = {}
        self._nid: Dict[object, int] = {}
        self._next = itertools.count()
        self._lock = threading.RLock()
        self._cb = _lib.PINNED_FN(self._pinned_cb)
        self._lookup = self._lib.tdkv_segidx_lookup
        self._one = ctypes.c_int64(-1)

    def __del__(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._lib.tdkv_segidx_destroy(h)

    # -- native plumbing ------------------------------------------------------
    def _pinned_cb(self, ctx, entry_id) -> int:
        return 1 if self._is_pinned(self._entries[int(entry_id)].kv_ref) else 0

    def _finish_evictions(self, ids: np.ndarray, n: int) -> int:
        for i in ids[:n]:
            entry = self._entries.pop(int(i))
            self._nid.pop(entry, None)
            if self._on_evict is not None:
                self._on_evict(entry)
        return n

    def _call(self, name: str, *args) -> None:
        rc = getattr(self._lib, name)(*args)
        if rc != 0:
            raise _lib.TdkvError(f"{name} failed ({rc}): "
                                 f"{self._lib.tdkv_last_error().decode(errors='replace')}")

    # -- reference API -----------------------------------------------------------
    def __len__(self) -> int:
        return int(self._lib.tdkv_segidx_count(self._h))

    def __contains__(self, digest: bytes) -> bool:
        with self._lock:
            out = np.empty(1, np.int64)
            self._call("tdkv_segidx_lookup", self._h, _digest16(digest), 1, 0,
                       out.ctypes.data)
            return int(out[0]) >= 0

    @property
    def total_bytes(self) -> int:
        return int(self._lib.tdkv_segidx_total(self._h))

    def entries(self) -> tuple:
        """Snapshot of live entries, least recently used first."""
        with self._lock:
            ids = np.empty(max(1, len(self._entries)), np.int64)
            n = ctypes.c_int64(0)
            self._call("tdkv_segidx_entries", self._h, ids.ctypes.data, ids.size,
                       ctypes.byref(n))
            return tuple(self._entries[int(i)] for i in ids[:n.value])

    def lookup(self, digest: bytes) -> Optional[SegmentCacheEntry]:
        """Most recent entry for the digest, or None. Refreshes recency."""
        with self._lock:
            out = self._one
            rc = self._lookup(self._h, _digest16(digest), 1, 1, ctypes.addressof(out))
            if rc:
                self._call("tdkv_segidx_lookup", self._h, _digest16(digest), 1, 1,
                           ctypes.addressof(out))
            return self._entries.get(out.value) if out.value >= 0 else None

    def lookup_many(self, digests: Sequence[bytes]) -> List[Optional[SegmentCacheEntry]]:
        """``lookup`` for a whole round in one native call (same recency
        effect as looking the digests up one by one, in order)."""
        with self._lock:
            n = len(digests)
            if n == 0:
                return []
            try:
                keys = b"".join(digests)
                if len(keys) != 16 * n:
                    raise TypeError
            except TypeError:
                keys = b"".join(_digest16(d) for d in digests)
            out = np.empty(n, np.int64)
            self._call("tdkv_segidx_lookup", self._h, keys, n, 1, out.ctypes.data)
            get = self._entries.get
            return [get(i) for i in out.tolist()]

    def insert(self, entry: SegmentCacheEntry) -> None:
        """Add an entry, then evict least-recently-used entries to budget."""
        with self._lock:
            if entry in self._nid:
                raise ValueError("entry is already in the index")
            nid = next(self._next)
            self._entries[nid] = entry
            self._nid[entry] = nid
            ids = np.empty(len(self._entries), np.int64)
            n = ctypes.c_int32(0)
            self._call("tdkv_segidx_insert", self._h, _digest16(entry.digest), nid,
                       int(entry.nbytes), self._cb, None, ids.ctypes.data, ids.size,
                       ctypes.byref(n))
            self._finish_evictions(ids, n.value)

    def remove(self, entry: SegmentCacheEntry) -> None:
        """Remove an entry (PinnedEntryError if pinned).  Like the reference
        (segment_index.py:172-181), removing an entry that is not in the
        index still subtracts its size and reports it to ``on_evict``."""
        with self._lock:
            if self._is_pinned(entry.kv_ref):
                raise PinnedEntryError("entry is pinned by live mirrors")
            nid = self._nid.pop(entry, -1)
            self._entries.pop(nid, None)
            self._call("tdkv_segidx_remove", self._h, nid, int(entry.nbytes))
            if self._on_evict is not None:
                self._on_evict(entry)

    def evict_to_budget(self, budget_bytes: Optional[int] = None) -> int:
        """Evict LRU-first down to the budget; returns entries removed.
        Pinned entries are skipped, so the total may stay above budget."""
        with self._lock:
            budget = self.budget_bytes if budget_bytes is None else int(budget_bytes)
            ids = np.empty(max(1, len(self._entries)), np.int64)
            n = ctypes.c_int32(0)
            self._call("tdkv_segidx_evict", self._h, budget, self._cb, None,
                       ids.ctypes.data, ids.size, ctypes.byref(n))
            return self._finish_evictions(ids, n.value)
