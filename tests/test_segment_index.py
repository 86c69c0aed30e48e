"""Native segment index (tdkv_segidx_*, host C++) against the reference's
behaviour: the reference's own test cases (pkg/tests/test_segment_index.py)
restated, plus a randomized operation stream checked step by step against
the oracle restatement.  Host-only code: runs without a GPU."""
import hashlib

import numpy as np
import pytest

from oracle import roundkv_port as ref
from paper_2604_03143_b200.segment_index import (EmptySegmentError, PinnedEntryError,
                                                 SegmentCacheEntry, SegmentIndex)


def digest(tokens):
    return hashlib.blake2b(np.asarray(tokens, dtype="<u4").tobytes(), digest_size=16).digest()


def entry(tokens, nbytes=100, src_start=0, ctx=b"c" * 16, ref_=None):
    return SegmentCacheEntry(digest(tokens), np.arange(src_start, src_start + len(tokens)), ref_,
                             ctx, nbytes)


def test_lookup_hits_regardless_of_source_offset():
    idx = SegmentIndex(budget_bytes=10_000)
    idx.insert(entry([4, 5, 6], src_start=10))
    hit = idx.lookup(digest([4, 5, 6]))
    assert hit is not None and hit.source_positions[0] == 10
    assert idx.lookup(digest([4, 5, 6])) is hit


def test_one_token_difference_is_a_distinct_entry():
    idx = SegmentIndex(budget_bytes=10_000)
    idx.insert(entry([1, 2, 3]))
    assert idx.lookup(digest([1, 2, 4])) is None
    assert idx.lookup(digest([1, 2, 3])) is not None


def test_lookup_returns_most_recent_for_digest():
    idx = SegmentIndex(budget_bytes=10_000)
    first, second = entry([9, 9], ctx=b"a" * 16), entry([9, 9], ctx=b"b" * 16)
    idx.insert(first)
    idx.insert(second)
    assert idx.lookup(digest([9, 9])) is second


def test_lru_eviction_under_budget_pressure():
    evicted = []
    idx = SegmentIndex(budget_bytes=250, on_evict=evicted.append)
    e1, e2, e3 = entry([1]), entry([2]), entry([3])
    idx.insert(e1)
    idx.insert(e2)
    idx.lookup(e1.digest)
    idx.insert(e3)
    assert evicted == [e2]
    assert idx.lookup(e2.digest) is None and idx.lookup(e1.digest) is e1
    assert idx.total_bytes == 200


def test_budget_zero_empties_unpinned_index():
    idx = SegmentIndex(budget_bytes=10_000)
    for t in range(5):
        idx.insert(entry([t]))
    assert idx.evict_to_budget(0) == 5
    assert len(idx) == 0 and idx.total_bytes == 0


def test_pinned_entries_survive_eviction():
    class Ref:
        def __init__(self, pinned):
            self.pinned = pinned

    idx = SegmentIndex(budget_bytes=10_000, is_pinned=lambda r: r.pinned)
    master, loose1, loose2 = entry([1], ref_=Ref(True)), entry([2], ref_=Ref(False)), \
        entry([3], ref_=Ref(False))
    for e in (master, loose1, loose2):
        idx.insert(e)
    idx.evict_to_budget(0)
    assert idx.lookup(master.digest) is master
    assert idx.lookup(loose1.digest) is None and idx.lookup(loose2.digest) is None
    assert idx.total_bytes == master.nbytes
    with pytest.raises(PinnedEntryError):
        idx.remove(master)
    master.kv_ref.pinned = False
    idx.evict_to_budget(0)
    assert len(idx) == 0


def test_entry_validation():
    with pytest.raises(EmptySegmentError):
        SegmentCacheEntry(b"d" * 16, np.array([], dtype=np.int64), None, b"c" * 16, 10)
    with pytest.raises(ValueError):
        SegmentCacheEntry(b"d" * 16, np.array([3, 2]), None, b"c" * 16, 10)
    with pytest.raises(ValueError):
        SegmentCacheEntry(b"d" * 16, np.array([1, 2]), None, b"c" * 16, 0)


def test_random_operation_stream_matches_oracle():
    """5,000 random inserts / lookups / lookup_many / removes / evictions with
    pins toggling, compared after every step with the oracle restatement of
    segment_index.py (lookup results, evicted entries in order, totals, LRU
    snapshot)."""
    rng = np.random.default_rng(17)

    class Ref:
        def __init__(self):
            self.pinned = False

    ev_a, ev_b = [], []
    a = SegmentIndex(2_000, is_pinned=lambda r: r.pinned, on_evict=ev_a.append)
    b = ref.SegmentIndexPort(2_000, is_pinned=lambda r: r.pinned, on_evict=ev_b.append)
    live = []
    for step in range(5000):
        op = rng.integers(0, 10)
        if op < 4:
            toks = [int(rng.integers(0, 30))]
            e = entry(toks, nbytes=int(rng.integers(1, 300)), ref_=Ref())
            a.insert(e)
            b.insert(e)
            live.append(e)
        elif op < 6:
            d = digest([int(rng.integers(0, 30))])
            assert a.lookup(d) is b.lookup(d)
        elif op == 6:
            ds = [digest([int(rng.integers(0, 30))]) for _ in range(5)]
            assert a.lookup_many(ds) == [b.lookup(d) for d in ds]
        elif op == 7 and live:
            e = live[int(rng.integers(0, len(live)))]
            e.kv_ref.pinned = not e.kv_ref.pinned
        elif op == 8 and live:
            e = live[int(rng.integers(0, len(live)))]
            if e.kv_ref.pinned:
                with pytest.raises(PinnedEntryError):
                    a.remove(e)
                with pytest.raises(Exception):
                    b.remove(e)
            elif e in a.entries():
                a.remove(e)
                b.remove(e)
        else:
            budget = int(rng.integers(0, 3000))
            assert a.evict_to_budget(budget) == b.evict_to_budget(budget)
        assert ev_a == ev_b, step
        assert a.total_bytes == b.total_bytes and len(a) == len(b)
        assert a.entries() == b.entries()
        assert all((d in a) == (d in b) for d in (digest([0]), digest([7])))


def test_native_index_reproduces_reference_stream():
    """The reference's own recorded stream (tests/golden/make_golden.py,
    1,500 operations), replayed on the native index."""
    import json
    import os
    from helpers import replay_segment_index
    G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))

    def make(tok, nbytes, kv_ref):
        return SegmentCacheEntry(digest([tok]), np.arange(1), kv_ref, b"c" * 16, nbytes)

    replay_segment_index(lambda b, p, ev: SegmentIndex(b, is_pinned=p, on_evict=ev), make,
                         G["segment_index"])
