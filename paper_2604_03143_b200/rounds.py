"""Synthetic All-Gather rounds of the benchmark shapes.

An agent's prompt is ``hist || SEP || seg_{pi(0)} || SEP || ... || seg_{pi(S-1)}``
(the flattened layout of core.PromptLayout, one separator between segments),
so T = hist + S * (seg_len + 1).  Segment s's master rows were produced at
source positions p_s .. p_s + seg_len - 1 with p_s ~ U[0, 8192) (seed 1) to
exercise large |delta|; agent i reads the segments in the order
rng(2 + i).permutation(S).  K/V values are N(0, 1) float32 (seed 0), bf16
configs round the same values.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from .collector import CollectJob, MasterArena


@dataclass(frozen=True)
class RoundSpec:
    name: str
    num_layers: int
    num_heads: int
    head_dim: int
    dtype: str                 # "f32" | "bf16"
    num_agents: int
    num_segments: int
    seg_len: int
    hist_len: int
    max_source: int = 8192
    sessions: int = 1          # independent groups; agents and segments split evenly
    strong: bool = False       # multi-GPU: total agents fixed and sharded (else per-GPU fixed)
    sub_batch: int = 0         # >0: a GPU's pool holds this many agents; its shard is
                               # collected in sub-batches (C5 at small GPU counts)

    @property
    def agents_per_session(self) -> int:
        return -(-self.num_agents // self.sessions)

    @property
    def total_segments(self) -> int:
        return self.sessions * self.num_segments

    def session_of(self, agent: int) -> int:
        return min(self.sessions - 1, agent // self.agents_per_session)

    @property
    def tokens_per_agent(self) -> int:
        return self.hist_len + self.num_segments * (self.seg_len + 1)

    @property
    def torch_dtype(self) -> torch.dtype:
        return torch.float32 if self.dtype == "f32" else torch.bfloat16

    @property
    def itemsize(self) -> int:
        return 4 if self.dtype == "f32" else 2

    @property
    def row_bytes(self) -> int:
        return self.num_heads * self.head_dim * self.itemsize

    @property
    def master_rows(self) -> int:
        return self.sessions * self.num_segments * self.seg_len

    @property
    def master_bytes(self) -> int:
        """M: K+V bytes of every shared segment master (read once)."""
        return 2 * self.num_layers * self.master_rows * self.row_bytes

    @property
    def session_master_bytes(self) -> int:
        return self.master_bytes // self.sessions

    def collector_bytes(self, agents: Optional[int] = None) -> int:
        """Algorithmic collector bytes: every master of the
        sessions the first ``agents`` agents belong to, read once, plus each
        agent's copy of its session's masters, written (M + N*M for one
        session)."""
        n = self.num_agents if agents is None else agents
        touched = len({self.session_of(a) for a in range(n)})
        return self.session_master_bytes * (touched + n)

    def collector_bytes_for(self, agents: Sequence[int]) -> int:
        """Algorithmic collector bytes of an arbitrary agent set: the masters
        of every session it touches read once, one copy written per agent."""
        agents = list(agents)
        touched = len({self.session_of(a) for a in agents})
        return self.session_master_bytes * (touched + len(agents))

    def session_rows(self, session: int) -> Tuple[int, int]:
        """Arena row range [r0, r1) of a session's masters."""
        n = self.num_segments * self.seg_len
        return session * n, (session + 1) * n

    def sessions_of(self, agents: Sequence[int]) -> List[int]:
        return sorted({self.session_of(a) for a in agents})

    @property
    def dense_bytes(self) -> int:
        return 2 * self.num_layers * self.tokens_per_agent * self.row_bytes

    def scaled(self, **kw) -> "RoundSpec":
        d = dict(self.__dict__)
        d.update(kw)
        return RoundSpec(**d)


CONFIGS = {
    "c1": RoundSpec("c1-toy-8x4x256-f32", 2, 8, 64, "f32", 8, 4, 256, 64),
    "c2": RoundSpec("c2-qwen7b-50x16x256-bf16", 28, 4, 128, "bf16", 50, 16, 256, 512),
    "c3": RoundSpec("c3-qwen14b-250x25x20-10sessions-bf16", 48, 8, 128, "bf16", 250, 25, 20,
                    192, sessions=10, strong=True),
    "c4": RoundSpec("c4-agentsociety-100x32x128-bf16", 28, 4, 128, "bf16", 100, 32, 128, 8192),
    "c5": RoundSpec("c5-qwen7b-1000-agent-shard-bf16", 28, 4, 128, "bf16", 1000, 16, 256, 512,
                    strong=True, sub_batch=125),
}


def source_offsets(spec: RoundSpec) -> np.ndarray:
    """Source position of every (global) segment's master."""
    return np.random.default_rng(1).integers(0, spec.max_source,
                                             spec.total_segments).astype(np.int64)


def agent_order(agent: int, num_segments: int) -> np.ndarray:
    return np.random.default_rng(2 + agent).permutation(num_segments)


def segment_starts(spec: RoundSpec, agent: int) -> np.ndarray:
    """Prompt offset of each of the agent's session segments (indexed by the
    segment's index within the session)."""
    order = agent_order(agent, spec.num_segments)
    starts = np.empty(spec.num_segments, np.int64)
    starts[order] = spec.hist_len + 1 + np.arange(spec.num_segments) * (spec.seg_len + 1)
    return starts


def master_planes_host(spec: RoundSpec, seed: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """(L, sessions*S*len, H, D) float32 masters, rows grouped by global segment."""
    g = torch.Generator().manual_seed(seed)
    shape = (spec.num_layers, spec.master_rows, spec.num_heads, spec.head_dim)
    k = torch.randn(shape, generator=g, dtype=torch.float32)
    v = torch.randn(shape, generator=g, dtype=torch.float32)
    return k.numpy(), v.numpy()


def make_arena(spec: RoundSpec, k, v) -> MasterArena:
    """Wrap (L, master_rows, H, D) device planes as the round's master arena."""
    src = source_offsets(spec)
    n = spec.total_segments
    return MasterArena(k, v, np.arange(n) * spec.seg_len, np.full(n, spec.seg_len),
                       [np.arange(p, p + spec.seg_len) for p in src])


def agent_jobs(spec: RoundSpec, agent: int, slots: np.ndarray) -> List[CollectJob]:
    """The collector jobs of one agent: segment s lands at its prompt rows."""
    starts = segment_starts(spec, agent)
    src = source_offsets(spec)
    base = spec.session_of(agent) * spec.num_segments
    jobs = []
    for s in range(spec.num_segments):
        t0 = int(starts[s])
        dst = slots[t0:t0 + spec.seg_len]
        g = base + s
        delta = np.full(spec.seg_len, t0 - int(src[g]), np.int64)
        jobs.append(CollectJob(g, dst, delta))
    return jobs


def agent_starts(spec: RoundSpec, agents) -> np.ndarray:
    """(n, S) prompt offsets of every agent's session segments: the round's
    prompt layouts (host metadata the round starts from)."""
    return np.stack([segment_starts(spec, a) for a in agents])


def round_offsets(spec: RoundSpec, agents, slot_base: np.ndarray,
                  starts: Optional[np.ndarray] = None):
    """Vectorized job arrays of a round for ``plan_offsets``: (global segment
    ids, destination offsets into the agents' slot arena, per-job delta);
    ``starts`` = agent_starts(spec, agents) when the layouts are at hand."""
    agents = list(agents)
    if starts is None:
        starts = agent_starts(spec, agents)                              # (n, S)
    sess = np.array([spec.session_of(a) for a in agents], np.int64)
    segs = (sess[:, None] * spec.num_segments + np.arange(spec.num_segments)).reshape(-1)
    src = source_offsets(spec)
    dst_off = (np.asarray(slot_base, np.int64)[:, None] + starts).reshape(-1)
    delta = (starts.reshape(-1) - src[segs])
    return segs, dst_off, delta


def shard(num_agents: int, rank: int, world: int) -> range:
    """Contiguous agent shard of a rank: sizes differ by at
    most one, so a session spans as few ranks as possible."""
    lo = rank * num_agents // world
    return range(lo, (rank + 1) * num_agents // world)


def session_owners(spec: RoundSpec, world: int) -> List[int]:
    """The rank holding each session's masters: the rank of the session's
    first agent (the masters are produced where that session runs)."""
    owners = []
    for s in range(spec.sessions):
        first = s * spec.agents_per_session
        owners.append(next(r for r in range(world) if first in shard(spec.num_agents, r, world)))
    return owners


def session_needs(spec: RoundSpec, world: int) -> List[List[int]]:
    """Per rank, the sessions whose masters its agent shard reads."""
    return [spec.sessions_of(shard(spec.num_agents, r, world)) for r in range(world)]


# ---------------------------------------------------------------------------
# toy-model recovery rounds (the caller of the Collector: collective_recover)


@dataclass
class ToyConfig:
    num_layers: int
    num_heads: int
    head_dim: int
    vocab_size: int
    rope_base: float = 10000.0


@dataclass
class ToyWeights:
    """Synthetic toy-transformer weights with the reference's shapes and
    distribution (U[-0.1, 0.1] float32; toymodel.py:36-57): ``embed`` (V, hid),
    ``wq/wk/wv/wm`` (L, hid, hid)."""

    config: ToyConfig
    embed: np.ndarray
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wm: np.ndarray


def toy_weights(num_layers: int, num_heads: int, head_dim: int, vocab_size: int,
                seed: int = 0) -> ToyWeights:
    rng = np.random.default_rng(seed)
    hid = num_heads * head_dim

    def u(*shape):
        return rng.uniform(-0.1, 0.1, size=shape).astype(np.float32)

    return ToyWeights(ToyConfig(num_layers, num_heads, head_dim, vocab_size), u(vocab_size, hid),
                      u(num_layers, hid, hid), u(num_layers, hid, hid), u(num_layers, hid, hid),
                      u(num_layers, hid, hid))


@dataclass(eq=False)
class ToyHit:
    """A shared segment resolved against the cache (pic.py:51-64)."""

    kv: object                  # LayeredKv of the segment master
    target_idx: np.ndarray

    @property
    def delta(self) -> np.ndarray:
        return self.target_idx - np.asarray(self.kv.positions, np.int64)

    def __len__(self) -> int:
        return int(self.target_idx.size)


@dataclass(eq=False)
class ToyRequest:
    """The fields of the reference's PreparedRequest (pic.py:67-98) that the
    recovery path reads."""

    request_id: int
    tokens: np.ndarray
    positions: np.ndarray
    private_idx: np.ndarray
    structural_idx: np.ndarray
    hits: list
    label_entry: np.ndarray
    label_offset: np.ndarray

    @property
    def num_tokens(self) -> int:
        return int(self.tokens.size)

    @property
    def shared_idx(self) -> np.ndarray:
        if not self.hits:
            return np.empty(0, dtype=np.int64)
        return np.sort(np.concatenate([h.target_idx for h in self.hits]))


@dataclass(eq=False)
class ToyGroup:
    members: list


def toy_round(weights: ToyWeights, num_agents: int = 8, num_segments: int = 4,
              seg_len: int = 256, hist_len: int = 64, separator: int = 0, seed: int = 0,
              device: Optional[torch.device] = None):
    """One All-Gather round of the toy model (BASELINE configs[0]: 8 agents x
    4 shared 256-token blocks).  Segment s is agent (s mod N)'s output,
    prefilled after that agent's history and a separator, so its master rows
    carry source positions hist+1 .. hist+seg_len; agent i's prompt is
    hist_i || SEP || seg_pi(0) || SEP || ... with pi = rng(2+i).permutation(S)
    (prepare_request's layout, pic.py:110-163).  Returns the members (one
    group: equal lengths, one digest set).  ``device``: keep the segment
    masters resident there (as a B200 deployment does) instead of host numpy
    planes like the reference's cache entries."""
    from .recompute import full_prefill
    rng = np.random.default_rng(seed)
    V = weights.config.vocab_size
    hists = [rng.integers(1, V, hist_len) for _ in range(num_agents)]
    outputs = [rng.integers(1, V, seg_len) for _ in range(num_segments)]
    segs = []
    for s in range(num_segments):
        producer = np.concatenate([hists[s % num_agents], [separator], outputs[s]])
        kv = full_prefill(weights, producer)
        lo = hist_len + 1
        k, v = kv.k[:, lo:].copy(), kv.v[:, lo:].copy()
        if device is not None:
            k, v = torch.from_numpy(k).to(device), torch.from_numpy(v).to(device)
        segs.append(type(kv)(k, v, kv.positions[lo:].copy()))
    members = []
    for i in range(num_agents):
        order = np.random.default_rng(2 + i).permutation(num_segments)
        toks = [hists[i]]
        T = hist_len
        starts = []
        for j, s in enumerate(order):
            toks += [[separator], outputs[s]]
            starts.append(T + 1)
            T += seg_len + 1
        tokens = np.concatenate(toks).astype(np.int64)
        label_entry = np.full(T, -1, np.int64)
        label_offset = np.full(T, -1, np.int64)
        hits = []
        for s, st in zip(order, starts):
            idx = np.arange(st, st + seg_len, dtype=np.int64)
            hits.append(ToyHit(segs[s], idx))
            label_entry[idx] = s
            label_offset[idx] = np.arange(seg_len)
        members.append(ToyRequest(i, tokens, np.arange(T, dtype=np.int64),
                                  np.arange(hist_len, dtype=np.int64),
                                  np.asarray([st - 1 for st in starts], np.int64), hits,
                                  label_entry, label_offset))
    return members


class _SeedRows:
    """The cached rows of a segment master as the index sees them (count
    and source positions; the planes live in the round's master arena)."""

    def __init__(self, positions: np.ndarray) -> None:
        self.positions = positions

    @property
    def num_tokens(self) -> int:
        return int(self.positions.size)


class _SeedRef:
    def __init__(self, kv) -> None:
        self.kv = kv


def round_layouts(spec: RoundSpec, agents, separator: int, seed: int = 7):
    """The round as the reference's objects: one PromptLayout per agent
    (private history, then the session's shared outputs in the agent's
    order -- the layout ``segment_starts`` describes) and a SegmentIndex
    holding every segment master at its source positions.  Returns
    (layouts, index, {id(entry): global segment})."""
    from .prepare import PromptLayout, Segment, SegmentKind
    from .segment_index import SegmentCacheEntry, SegmentIndex
    rng = np.random.default_rng(seed)
    vocab = max(2, separator)
    shared = [Segment(tuple(rng.integers(0, vocab, spec.seg_len).tolist()),
                      SegmentKind.SHARED_OUTPUT) for _ in range(spec.total_segments)]
    index = SegmentIndex(1 << 62)
    src = source_offsets(spec)
    entry_segment = {}
    for g, seg in enumerate(shared):
        pos = np.arange(src[g], src[g] + spec.seg_len, dtype=np.int64)
        e = SegmentCacheEntry(seg.digest, pos, _SeedRef(_SeedRows(pos)), b"",
                              2 * spec.num_layers * spec.seg_len * spec.row_bytes)
        index.insert(e)
        entry_segment[id(e)] = g
    layouts = []
    for a in agents:
        hist = Segment(tuple(rng.integers(0, vocab, spec.hist_len).tolist()),
                       SegmentKind.PRIVATE_HISTORY)
        base = spec.session_of(a) * spec.num_segments
        order = agent_order(a, spec.num_segments)
        layouts.append(PromptLayout(a, (hist,) + tuple(shared[base + s] for s in order)))
    return layouts, index, entry_segment
