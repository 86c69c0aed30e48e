"""Request preparation for a round, in native code.

Drop-in for the reference's ``pic.prepare_request`` (pic.py:110-163) and the
prompt types it reads (core.py:17-140: ``SegmentKind``, ``Segment``,
``PromptLayout``, ``token_digest``, ``flatten_prompt``).  The per-prompt
work -- flattening with separators, resolving SHARED_OUTPUT segments in the
segment index, labelling hit positions with (entry id, offset), collecting
the structural-fresh positions -- runs in C++ (``tdkv_prepare_batch``) for
all prompts of a round at once: a round's prompts share their shared-output
segments, so each distinct segment's tokens are converted once and every
prompt is a list of segment ids.  ``prepare_request`` is the batch of one.

``plan_offsets_from_prepared`` turns the prepared requests of a round into
the collector's job arrays (segment, destination offset into the agents'
slot arena, delta) -- the host planning between the reference objects and
``KVCollector.plan_offsets``.

Layouts of the reference's own classes work too: segments are read through
``.tokens``, ``.kind`` (an enum whose ``.value`` is "private_history",
"shared_output" or "round_task") and ``.digest``.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from enum import Enum
from typing import List, Optional, Sequence

import numpy as np

from . import _lib


class SegmentKind(Enum):
    PRIVATE_HISTORY = "private_history"
    SHARED_OUTPUT = "shared_output"
    ROUND_TASK = "round_task"


_KIND_CODE = {"private_history": 0, "shared_output": 1, "round_task": 2}


def token_digest(tokens: Sequence[int]) -> bytes:
    """128-bit content digest of a token sequence (core.py:23-30)."""
    raw = np.asarray(tokens, dtype="<u4").tobytes()
    return hashlib.blake2b(raw, digest_size=16).digest()


@dataclass(frozen=True)
class Segment:
    """A separator-free run of tokens with a content digest (core.py:70-87)."""

    tokens: tuple
    kind: SegmentKind
    digest: bytes = field(init=False, repr=False)

    def __post_init__(self) -> None:
        toks = tuple(int(t) for t in self.tokens)
        if len(toks) == 0:
            raise ValueError("segment must contain at least one token")
        if any(t < 0 for t in toks):
            raise ValueError("token ids must be non-negative")
        object.__setattr__(self, "tokens", toks)
        object.__setattr__(self, "digest", token_digest(toks))

    def __len__(self) -> int:
        return len(self.tokens)


@dataclass(frozen=True)
class PromptLayout:
    """Ordered segments of one request's prompt (core.py:90-127)."""

    agent_id: int
    segments: tuple

    def __post_init__(self) -> None:
        segs = tuple(self.segments)
        if not segs:
            raise ValueError("prompt needs at least one segment")
        private = [i for i, s in enumerate(segs) if s.kind is SegmentKind.PRIVATE_HISTORY]
        if len(private) != 1 or private[0] != 0:
            raise ValueError("exactly one private-history segment, and it must be first")
        object.__setattr__(self, "segments", segs)

    @property
    def total_len(self) -> int:
        return sum(len(s) for s in self.segments)

    @property
    def flat_len(self) -> int:
        return self.total_len + len(self.segments) - 1

    def segment_starts(self) -> list:
        starts, pos = [], 0
        for seg in self.segments:
            starts.append(pos)
            pos += len(seg) + 1
        return starts


def flatten_prompt(layout, separator: int) -> list:
    """Join segments with single separators (core.py:130-140)."""
    for seg in layout.segments:
        if separator in seg.tokens:
            raise ValueError("separator id must not occur inside a segment")
    out: list = []
    for i, seg in enumerate(layout.segments):
        if i:
            out.append(int(separator))
        out.extend(seg.tokens)
    return out


@dataclass(eq=False)
class HitSegment:
    """A shared segment resolved against the cache (pic.py:51-64)."""

    entry: object
    kv: object
    target_idx: np.ndarray

    @property
    def delta(self) -> np.ndarray:
        return self.target_idx - self.entry.source_positions

    def __len__(self) -> int:
        return int(self.target_idx.size)


@dataclass(eq=False)
class PreparedRequest:
    """A request with its hit/miss classification snapshotted (pic.py:67-98)."""

    request_id: int
    layout: object
    tokens: np.ndarray
    positions: np.ndarray
    private_idx: np.ndarray
    structural_idx: np.ndarray
    hits: list
    slot_map: object = None
    label_entry: np.ndarray = field(default=None, repr=False)
    label_offset: np.ndarray = field(default=None, repr=False)

    @property
    def num_tokens(self) -> int:
        return int(self.tokens.size)

    @property
    def shared_idx(self) -> np.ndarray:
        if not self.hits:
            return np.empty(0, dtype=np.int64)
        return np.sort(np.concatenate([h.target_idx for h in self.hits]))

    @property
    def hit_digests(self) -> frozenset:
        return frozenset(h.entry.digest for h in self.hits)


def _kind_code(kind) -> int:
    v = getattr(kind, "value", kind)
    try:
        return _KIND_CODE[v]
    except KeyError:
        raise ValueError(f"unknown segment kind {kind!r}") from None


@dataclass
class PreparedBatch:
    """The flat native outputs of a round (kept alive by the requests' views)."""

    tok_off: np.ndarray
    tokens: np.ndarray
    label_entry: np.ndarray
    label_offset: np.ndarray
    struct_off: np.ndarray
    structural: np.ndarray
    private_len: np.ndarray
    hits: np.ndarray             # (n_hits, 4): prompt segment index, entry id, target start, len
    hit_off: np.ndarray
    hit_entries: list            # SegmentCacheEntry per hit


def prepare_batch(layouts: Sequence, separator: int, cache, threads: int = 0) -> PreparedBatch:
    """The native preparation of a round's prompts (tdkv_prepare_batch)."""
    lib = _lib.load()
    seg_id: dict = {}
    seg_objs: list = []
    prompt_seg = []
    prompt_off = [0]
    for lay in layouts:
        for seg in lay.segments:
            k = id(seg)
            s = seg_id.get(k)
            if s is None:
                s = seg_id[k] = len(seg_objs)
                seg_objs.append(seg)
            prompt_seg.append(s)
        prompt_off.append(len(prompt_seg))
    n_segs = len(seg_objs)
    kinds = np.fromiter((_kind_code(s.kind) for s in seg_objs), np.int32, n_segs)
    lens = np.fromiter((len(s.tokens) for s in seg_objs), np.int64, n_segs)
    seg_tok_off = np.zeros(n_segs + 1, np.int64)
    np.cumsum(lens, out=seg_tok_off[1:])
    seg_tokens = np.empty(int(seg_tok_off[-1]), np.int64)
    for s, seg in enumerate(seg_objs):
        toks = seg.tokens
        seg_tokens[seg_tok_off[s]:seg_tok_off[s + 1]] = (
            toks if isinstance(toks, np.ndarray) else np.fromiter(toks, np.int64, len(toks)))
    digests = np.frombuffer(b"".join(
        s.digest if kinds[i] == 1 else b"\0" * 16 for i, s in enumerate(seg_objs)),
        np.uint8) if n_segs else np.zeros(0, np.uint8)
    if kinds.size and ((kinds == 1) & (np.fromiter((len(s.digest) for s in seg_objs), np.int64,
                                                   n_segs) != 16)).any():
        from .segment_index import _digest16
        digests = np.frombuffer(b"".join(_digest16(s.digest) if kinds[i] == 1 else b"\0" * 16
                                         for i, s in enumerate(seg_objs)), np.uint8)
    prompt_off = np.asarray(prompt_off, np.int32)
    prompt_seg = np.asarray(prompt_seg, np.int32)
    n_prompts = len(layouts)
    # output sizes: flat tokens and the structural capacity (all non-private
    # tokens + separators) follow from the inputs
    seg_of = lens[prompt_seg] if prompt_seg.size else np.zeros(0, np.int64)
    first = np.zeros(prompt_seg.size, bool)
    first[prompt_off[:-1][prompt_off[:-1] < prompt_seg.size]] = True
    total = int(seg_of.sum()) + int(prompt_seg.size - n_prompts)
    cap = int(seg_of[~first].sum()) + int(prompt_seg.size - n_prompts)
    n_shared = int((kinds[prompt_seg] == 1).sum()) if prompt_seg.size else 0
    # native id -> entry id table of the index (label_entry holds entry ids)
    ent = cache._entries if cache is not None else {}
    n_nid = (max(ent) + 1) if ent else 0
    nid_entry = np.full(max(1, n_nid), -1, np.int64)
    for nid, e in ent.items():
        nid_entry[nid] = e.entry_id
    out = PreparedBatch(np.empty(n_prompts + 1, np.int64), np.empty(max(1, total), np.int64),
                        np.empty(max(1, total), np.int64), np.empty(max(1, total), np.int64),
                        np.empty(n_prompts + 1, np.int64), np.empty(max(1, cap), np.int64),
                        np.zeros(max(1, n_prompts), np.int64),
                        np.empty((max(1, n_shared), 4), np.int64),
                        np.empty(n_prompts + 1, np.int64), [])
    hit_nid = np.empty(max(1, n_shared), np.int64)
    handle = cache._h if cache is not None else None
    lock = cache._lock if cache is not None else None
    d = lambda a: a.ctypes.data    # noqa: E731
    if lock is not None:
        lock.acquire()
    try:
        rc = lib.tdkv_prepare_batch(handle, n_prompts, d(prompt_off), d(prompt_seg), n_segs,
                                    d(kinds), d(seg_tok_off), d(seg_tokens), d(digests),
                                    int(separator), d(nid_entry), n_nid, d(out.tok_off),
                                    d(out.tokens), d(out.label_entry), d(out.label_offset),
                                    d(out.struct_off), d(out.structural), d(out.private_len),
                                    d(out.hits), d(out.hit_off), d(hit_nid), int(threads))
    finally:
        if lock is not None:
            lock.release()
    if rc:
        msg = lib.tdkv_last_error().decode(errors="replace")
        raise ValueError(msg.split(": ", 1)[1] if msg.startswith("segment ") or
                         msg.startswith("prompt ") else msg)
    nh = int(out.hit_off[-1])
    out.hits = out.hits[:nh]
    out.hit_entries = [ent[int(i)] for i in hit_nid[:nh]]
    return out


def _check_entry(entry, n: int) -> None:
    kv = entry.kv_ref.kv
    if kv.num_tokens != n or not np.array_equal(kv.positions, entry.source_positions):
        raise ValueError("cache entry does not cover its segment")


def prepare_requests(layouts: Sequence, model, cache, request_ids: Optional[Sequence[int]] = None,
                     slot_maps: Optional[Sequence] = None, threads: int = 0
                     ) -> List[PreparedRequest]:
    """prepare_request (pic.py:110-163) for every prompt of a round in one
    native pass; the requests' arrays are views of the batch outputs."""
    n = len(layouts)
    ids = list(range(n)) if request_ids is None else list(request_ids)
    maps = [None] * n if slot_maps is None else list(slot_maps)
    b = prepare_batch(layouts, model.separator_token, cache, threads)
    checked = set()
    out = []
    for p, lay in enumerate(layouts):
        t0, t1 = int(b.tok_off[p]), int(b.tok_off[p + 1])
        s0, s1 = int(b.struct_off[p]), int(b.struct_off[p + 1])
        hits = []
        for h in range(int(b.hit_off[p]), int(b.hit_off[p + 1])):
            _seg, _eid, start, ln = (int(x) for x in b.hits[h])
            entry = b.hit_entries[h]
            if id(entry) not in checked:
                _check_entry(entry, ln)
                checked.add(id(entry))
            hits.append(HitSegment(entry, entry.kv_ref.kv,
                                   np.arange(start, start + ln, dtype=np.int64)))
        out.append(PreparedRequest(
            request_id=ids[p], layout=lay, tokens=b.tokens[t0:t1],
            positions=np.arange(t1 - t0, dtype=np.int64),
            private_idx=np.arange(int(b.private_len[p]), dtype=np.int64),
            structural_idx=b.structural[s0:s1], hits=hits, slot_map=maps[p],
            label_entry=b.label_entry[t0:t1], label_offset=b.label_offset[t0:t1]))
    return out


def prepare_request(layout, model, cache, request_id: int = 0,
                    slot_map: object = None) -> PreparedRequest:
    """Drop-in for pic.prepare_request (pic.py:110-163)."""
    return prepare_requests([layout], model, cache, [request_id], [slot_map])[0]


def plan_offsets_from_prepared(batch: PreparedBatch, entry_segment: dict,
                               slot_base: np.ndarray):
    """The collector's job arrays of a prepared round: for every hit, the
    arena segment of its entry, the destination offset of its first token in
    the agents' slot arena (slot_base[prompt] + target start) and its delta
    (target start - the entry's first source position; the entry's source
    positions must be contiguous).  Vectorized over the whole round."""
    nh = batch.hits.shape[0]
    for e in {id(e): e for e in batch.hit_entries}.values():
        src = np.asarray(e.source_positions)
        if int(src[-1]) - int(src[0]) != src.size - 1:
            raise ValueError("offset planning needs contiguous source positions")
    prompt = np.repeat(np.arange(batch.hit_off.size - 1, dtype=np.int64),
                       np.diff(batch.hit_off))
    src0 = np.fromiter((e.source_positions[0] for e in batch.hit_entries), np.int64, nh)
    segs = np.fromiter((entry_segment[id(e)] for e in batch.hit_entries), np.int64, nh)
    start = batch.hits[:, 2]
    dst_off = np.asarray(slot_base, np.int64)[prompt] + start
    return segs, dst_off, start - src0
