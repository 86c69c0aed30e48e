"""Native request preparation (tdkv_prepare_batch behind
paper_2604_03143_b200.prepare) against the reference's prepare_request
(pic.py:110-163) outputs recorded by tests/golden/make_golden.py -- the
oracle restatement first, then the native batch -- plus the segment index's
recency and eviction afterwards.  Host-only: runs without a GPU."""
import numpy as np
import pytest

from helpers import load_golden, load_npz
from oracle import roundkv_port as ref
from paper_2604_03143_b200 import prepare as pp
from paper_2604_03143_b200.segment_index import SegmentCacheEntry, SegmentIndex
from paper_2604_03143_b200.core import LayeredKv

G = load_golden()
KIND = {"P": pp.SegmentKind.PRIVATE_HISTORY, "T": pp.SegmentKind.ROUND_TASK}


class _Ref:
    def __init__(self, kv):
        self.kv = kv


def _world():
    g = G["prepare"]
    segs = {n: pp.Segment(tuple(t), KIND.get(n[0], pp.SegmentKind.SHARED_OUTPUT))
            for n, t in g["tokens"].items()}
    return g, segs


def _index(g, segs, port=False):
    index = ref.SegmentIndexPort(10_000) if port else SegmentIndex(10_000)
    name_of = {}
    for name, seg, src in g["entries"]:
        n = len(segs[seg])
        kv = LayeredKv(np.zeros((1, n, 1, 2), np.float32), np.zeros((1, n, 1, 2), np.float32),
                       np.arange(src, src + n))
        e = SegmentCacheEntry(segs[seg].digest, kv.positions, _Ref(kv), b"ctx", 1000)
        index.insert(e)
        name_of[e.entry_id] = name
    return index, name_of


def _check(prep_like, want, name_of):
    assert prep_like["tokens"] == want["tokens"]
    assert prep_like["private_idx"] == want["private_idx"]
    assert prep_like["structural_idx"] == want["structural_idx"]
    assert prep_like["label_offset"] == want["label_offset"]
    assert [name_of.get(int(e)) for e in prep_like["label_entry"]] == want["label_entry"]
    assert prep_like["hits"] == want["hits"]


def test_oracle_prepare_matches_reference():
    g, segs = _world()
    index, name_of = _index(g, segs, port=True)
    for names, want in zip(g["prompts"], g["requests"]):
        p = ref.prepare_request_port([(segs[n].kind.value, segs[n].tokens, segs[n].digest)
                                      for n in names], g["separator"], index.lookup)
        _check({"tokens": p.tokens.tolist(), "private_idx": p.private_idx.tolist(),
                "structural_idx": p.structural_idx.tolist(),
                "label_offset": p.label_offset.tolist(), "label_entry": p.label_entry.tolist(),
                "hits": [[name_of[e.entry_id], t.tolist(), (t - e.source_positions).tolist()]
                         for e, t in p.hits]}, want, name_of)
    assert [name_of[e.entry_id] for e in index.entries()] == g["recency"]


class _Model:
    def __init__(self, sep):
        self.separator_token = sep


@pytest.mark.parametrize("batched", [True, False])
def test_native_prepare_matches_reference(batched):
    g, segs = _world()
    index, name_of = _index(g, segs)
    layouts = [pp.PromptLayout(i, tuple(segs[n] for n in names))
               for i, names in enumerate(g["prompts"])]
    model = _Model(g["separator"])
    if batched:
        preps = pp.prepare_requests(layouts, model, index)
    else:
        preps = [pp.prepare_request(lay, model, index, request_id=i)
                 for i, lay in enumerate(layouts)]
    for p, want in zip(preps, g["requests"]):
        _check({"tokens": p.tokens.tolist(), "private_idx": p.private_idx.tolist(),
                "structural_idx": p.structural_idx.tolist(),
                "label_offset": p.label_offset.tolist(), "label_entry": p.label_entry.tolist(),
                "hits": [[name_of[h.entry.entry_id], h.target_idx.tolist(), h.delta.tolist()]
                         for h in p.hits]}, want, name_of)
        assert p.positions.tolist() == list(range(p.num_tokens))
    # lookups refreshed recency in prompt / segment order, exactly as the
    # reference's one-by-one lookups: same LRU order, same eviction
    assert [name_of[e.entry_id] for e in index.entries()] == g["recency"]
    evicted = []
    index._on_evict = lambda e: evicted.append(name_of[e.entry_id])
    n = len(segs["A"])
    kv = LayeredKv(np.zeros((1, n, 1, 2), np.float32), np.zeros((1, n, 1, 2), np.float32),
                   np.arange(n))
    index.insert(SegmentCacheEntry(b"x" * 16, kv.positions, _Ref(kv), b"ctx", 7000))
    assert evicted == g["evicted_after_insert"]


def test_native_prepare_errors():
    g, segs = _world()
    index, _ = _index(g, segs)
    bad = pp.PromptLayout(9, (segs["P0"], segs["A"]))
    with pytest.raises(ValueError) as err:
        pp.prepare_request(bad, _Model(segs["A"].tokens[0]), index)
    assert str(err.value) == g["separator_error"]
    # an entry whose cached rows do not cover the segment
    kv = LayeredKv(np.zeros((1, 2, 1, 2), np.float32), np.zeros((1, 2, 1, 2), np.float32),
                   np.arange(2))
    index.insert(SegmentCacheEntry(segs["M"].digest, kv.positions, _Ref(kv), b"ctx", 10))
    with pytest.raises(ValueError, match="does not cover"):
        pp.prepare_request(pp.PromptLayout(0, (segs["P1"], segs["M"])), _Model(511), index)


def test_native_prepare_reproduces_t3_requests():
    """The reference's T3 rounds (tests/golden/t3.npz): every prepared
    request of both rounds, rebuilt natively from its recorded layout against
    an index seeded like trace._seed_path (trace.py:176-181)."""
    z = load_npz("t3.npz")
    for case, meta in G["t3"].items():
        index = SegmentIndex(64 * 1024 * 1024)
        seed_of = {}
        model = _Model(meta["model"][3] - 1)
        for rmeta in meta["rounds"]:
            for key in rmeta["seeds"]:
                pos = z[key + "_pos"]
                kv = LayeredKv(z[key + "_k"], z[key + "_v"], pos)
                e = SegmentCacheEntry(pp.token_digest(z[key + "_tokens"].tolist()), pos, _Ref(kv),
                                      b"ctx", kv.dense_nbytes)
                index.insert(e)
                seed_of[e.entry_id] = key
            reqs = [m for g in rmeta["groups"] for m in g["members"]] + rmeta["remainder"]
            reqs.sort(key=lambda m: m["agent"])
            layouts = []
            for m in reqs:
                tag = m["tag"]
                kinds, lens = z[f"{tag}_layout_kinds"], z[f"{tag}_layout_lens"]
                toks = np.split(z[f"{tag}_layout_tokens"], np.cumsum(lens)[:-1])
                layouts.append(pp.PromptLayout(m["agent"], tuple(
                    pp.Segment(tuple(t.tolist()), pp.SegmentKind(k)) for k, t in zip(kinds, toks))))
            preps = pp.prepare_requests(layouts, model, index, [m["rid"] for m in reqs])
            for m, p in zip(reqs, preps):
                tag = m["tag"]
                for name in ("tokens", "positions", "private_idx", "structural_idx",
                             "label_offset"):
                    assert np.array_equal(getattr(p, name), z[f"{tag}_{name}"]), (tag, name)
                labels = [seed_of.get(int(e), "") for e in p.label_entry]
                assert labels == z[f"{tag}_label_seed"].tolist(), tag
                assert [[seed_of[h.entry.entry_id], h.target_idx.tolist()] for h in p.hits] == \
                    [[h["seed"], h["target"]] for h in m["hits"]]


def test_plan_offsets_from_prepared():
    g, segs = _world()
    index, name_of = _index(g, segs)
    layouts = [pp.PromptLayout(i, tuple(segs[n] for n in names))
               for i, names in enumerate(g["prompts"])]
    batch = pp.prepare_batch(layouts, g["separator"], index)
    entry_seg = {id(e): i for i, e in enumerate(index.entries())}
    base = np.array([100, 500, 900], np.int64)
    segs_, dst, delta = pp.plan_offsets_from_prepared(batch, entry_seg, base)
    want = []
    for p, req in enumerate(g["requests"]):
        for name, target, d in req["hits"]:
            want.append((base[p] + target[0], d[0]))
    assert list(zip(dst.tolist(), delta.tolist())) == want
    assert [name_of[index.entries()[s].entry_id] for s in segs_] == \
        [h[0] for r in g["requests"] for h in r["hits"]]


def test_round_planning_from_layouts_equals_synthetic_offsets():
    """The bench's host planning path (reference objects -> native prepare ->
    collector job arrays) yields exactly the jobs the synthetic round
    generator plans directly (rounds.round_offsets), for a multi-session
    round: same (segment, destination offset, delta) multiset."""
    from paper_2604_03143_b200 import rounds
    spec = rounds.CONFIGS["c3"].scaled(num_agents=30, num_layers=2)
    agents = list(range(30))
    layouts, index, eseg = rounds.round_layouts(spec, agents, 1023)
    batch = pp.prepare_batch(layouts, 1023, index)
    base = np.arange(30, dtype=np.int64) * spec.tokens_per_agent * 2
    got = pp.plan_offsets_from_prepared(batch, eseg, base)
    want = rounds.round_offsets(spec, agents, base)
    og, ow = np.lexsort((got[0], got[1])), np.lexsort((want[0], want[1]))
    for a, b in zip(got, want):
        assert np.array_equal(a[og], b[ow])
    assert batch.tok_off[-1] == 30 * spec.tokens_per_agent
