"""End-to-end recovery on the GPU (Collector K1 + selective recompute K5 +
selection K4) against the reference's own collective_recover /
recover_prepared outputs (tests/golden/recovery.npz)."""
import numpy as np
import pytest

from helpers import load_golden, load_npz
from oracle import roundkv_port as ref
from paper_2604_03143_b200 import pic
from paper_2604_03143_b200.core import LayeredKv
from paper_2604_03143_b200.ledger import CostLedger

pytestmark = pytest.mark.gpu
G = load_golden()["recovery"]
TOL = 1e-5


class _Cfg:
    def __init__(self, L, H, D, V):
        self.num_layers, self.num_heads, self.head_dim, self.vocab_size = L, H, D, V
        self.rope_base = 10000.0


class _Weights:
    def __init__(self, L, H, D, V, seed):
        w = ref.build_weights(L, H, D, V, seed)
        self.config = _Cfg(L, H, D, V)
        self.embed, self.wq, self.wk, self.wv, self.wm = w.embed, w.wq, w.wk, w.wv, w.wm


class _Hit:
    def __init__(self, kv, target):
        self.kv = kv
        self.target_idx = np.asarray(target, np.int64)
        self.delta = self.target_idx - kv.positions

    def __len__(self):
        return int(self.target_idx.size)


class _Prep:
    def __init__(self, z, case, m, segs):
        rid = m["rid"]
        self.request_id = rid
        for name in ("tokens", "positions", "private_idx", "structural_idx", "label_entry",
                     "label_offset"):
            setattr(self, name, z[f"{case}_r{rid}_{name}"])
        self.hits = [_Hit(segs[h["seg"]], h["target"]) for h in m["hits"]]

    @property
    def num_tokens(self):
        return int(self.tokens.size)

    @property
    def shared_idx(self):
        if not self.hits:
            return np.empty(0, dtype=np.int64)
        return np.sort(np.concatenate([h.target_idx for h in self.hits]))


class _Pic:
    recompute_fraction = 0.15
    check_layer = 1


def _world(case):
    z = load_npz("recovery.npz")
    meta = G[case]
    segs = [LayeredKv(z[f"{case}_seg{a}_k"], z[f"{case}_seg{a}_v"], z[f"{case}_seg{a}_pos"])
            for a in range(meta["agents"])]
    preps = [_Prep(z, case, m, segs) for m in meta["members"]]
    return z, meta, preps, _Weights(*meta["model"])


@pytest.mark.parametrize("case", ["same_order", "permuted"])
def test_collective_recover_matches_reference(case):
    z, meta, preps, w = _world(case)
    group = type("G", (), {"members": preps})
    led = CostLedger(3)
    results, plan = pic.collective_recover(w, group, _Pic, led)
    assert led.rope_calls_by_layer == [1, 1, 1] and led.selection_passes == 1
    assert plan.master_id == meta["master_id"]
    for m in meta["members"]:
        rid = m["rid"]
        r = results[rid]
        assert r.important_positions.tolist() == m["important"]
        assert abs(r.deviation_score - m["deviation"]) <= 1e-5 * max(1.0, abs(m["deviation"]))
        assert r.num_recomputed == m["num_recomputed"]
        assert np.abs(r.kv.k.cpu().numpy() - z[f"{case}_r{rid}_k"]).max() <= TOL
        assert np.abs(r.kv.v.cpu().numpy() - z[f"{case}_r{rid}_v"]).max() <= TOL
        if m["hints"] is not None:
            assert plan.mirror_diff_hints[rid].tolist() == m["hints"]


def test_serial_recovery_matches_reference():
    z, meta, preps, w = _world("permuted")
    led = CostLedger(3)
    r = pic.recover_prepared(w, preps[0], _Pic, led)
    assert led.rope_calls_by_layer == [1, 1, 1] and led.selection_passes == 1
    assert np.abs(r.kv.k.cpu().numpy() - z["permuted_serial0_k"]).max() <= TOL
    assert np.abs(r.kv.v.cpu().numpy() - z["permuted_serial0_v"]).max() <= TOL


@pytest.mark.parametrize("agents", [2, 3, 5, 10])
def test_grouped_equals_serial_across_group_sizes(agents):
    """Acceptance C01 (test_acceptance.py:80-114) on the GPU over group sizes
    {2, 3, 5, 10}: grouped == serial bit for bit, one rotation per layer."""
    import torch
    from paper_2604_03143_b200 import rounds
    w = rounds.toy_weights(3, 2, 16, 512, seed=agents)
    members = rounds.toy_round(w, num_agents=agents, num_segments=3, seg_len=24, hist_len=10,
                               seed=100 + agents)
    led = CostLedger(3)
    results, plan = pic.collective_recover(w, rounds.ToyGroup(members), _Pic, led)
    assert led.rope_calls_per_layer == 1 and led.selection_passes == 1
    for m in members:
        r = pic.recover_prepared(w, m, _Pic)
        g = results[m.request_id]
        assert torch.equal(g.kv.k, r.kv.k) and torch.equal(g.kv.v, r.kv.v)
        assert g.important_positions.tolist() == r.important_positions.tolist()
        assert g.deviation_score == r.deviation_score


def test_grouped_equals_serial_on_a_c1_round():
    """BASELINE configs[0] (8 agents x 4 shared 256-token blocks, 2-layer toy
    model, 8 heads, d=64): grouped recovery is bit-identical to serial
    recovery of every member -- caches, important sets, deviation scores
    (the reference's acceptance C01, test_acceptance.py:80-114) -- with one
    rotation and one selection pass per layer instead of one per member (C02)."""
    import torch
    from paper_2604_03143_b200 import rounds
    w = rounds.toy_weights(2, 8, 64, 1024, seed=3)
    members = rounds.toy_round(w, seed=5)
    led_g, led_s = CostLedger(2), CostLedger(2)
    results, plan = pic.collective_recover(w, rounds.ToyGroup(members), _Pic, led_g)
    for m in members:
        r = pic.recover_prepared(w, m, _Pic, led_s)
        g = results[m.request_id]
        assert torch.equal(g.kv.k, r.kv.k) and torch.equal(g.kv.v, r.kv.v)
        assert g.important_positions.tolist() == r.important_positions.tolist()
        assert g.deviation_score == r.deviation_score
        assert plan.deviation_scores[m.request_id] == r.deviation_score
    assert led_g.rope_calls_per_layer == 1
    assert led_s.rope_calls_per_layer == len(members)
    assert led_g.selection_passes == 1 and led_s.selection_passes == len(members)
    assert plan.master_id == min(plan.deviation_scores.items(), key=lambda kv: (kv[1], kv[0]))[0]


def test_segment_reuse_is_position_independent():
    """Acceptance C08 (test_acceptance.py:335-361) on the GPU: a segment
    produced at offset 10 is reused at offset 400 of another prompt; with
    recompute fraction 1 the recovered cache equals a full prefill of that
    prompt (GPU prefill within 1e-6, the oracle's within the model tolerance)."""
    import torch
    from paper_2604_03143_b200 import recompute, rounds
    w = rounds.toy_weights(4, 2, 8, 1024, seed=9)
    rng = np.random.default_rng(88)
    segment = rng.integers(1, 1024, 16)
    producer = np.concatenate([rng.integers(1, 1024, 9), [0], segment])
    consumer = np.concatenate([rng.integers(1, 1024, 399), [0], segment])
    kv = recompute.full_prefill(w, producer)
    seg_kv = type(kv)(kv.k[:, 10:].copy(), kv.v[:, 10:].copy(), kv.positions[10:].copy())
    assert seg_kv.positions[0] == 10
    T = consumer.size
    target = np.arange(400, 416, dtype=np.int64)
    le = np.full(T, -1, np.int64)
    lo = np.full(T, -1, np.int64)
    le[target], lo[target] = 0, np.arange(16)
    prep = rounds.ToyRequest(0, consumer.astype(np.int64), np.arange(T, dtype=np.int64),
                             np.arange(399, dtype=np.int64), np.array([399], np.int64),
                             [rounds.ToyHit(seg_kv, target)], le, lo)

    class _Full:
        recompute_fraction = 1.0
        check_layer = 1
    res = pic.recover_prepared(w, prep, _Full, CostLedger(4))
    full = recompute.full_prefill(w, consumer)
    got_k = res.kv.k.cpu().numpy()
    got_v = res.kv.v.cpu().numpy()
    assert np.abs(got_k - full.k).max() <= 1e-6 and np.abs(got_v - full.v).max() <= 1e-6
    ow = ref.ToyWeights(2, 8, 10000.0, w.embed, w.wq, w.wk, w.wv, w.wm)
    ok, ov = ref.full_prefill(ow, consumer)
    assert np.abs(got_k - ok).max() <= TOL and np.abs(got_v - ov).max() <= TOL


def _reuse_request(w, consumer_hist, segments):
    """A one-member request reading ``segments`` [(tokens, producer history)]
    after ``consumer_hist``; each segment's master is its producer's prefill
    (history || SEP || segment), i.e. cached at offset len(history) + 1."""
    from paper_2604_03143_b200 import recompute, rounds
    toks = [np.asarray(consumer_hist, np.int64)]
    T = len(consumer_hist)
    hits, structural = [], []
    le, lo = [], []
    for e, (seg, hist) in enumerate(segments):
        kv = recompute.full_prefill(w, np.concatenate([hist, [0], seg]))
        a = len(hist) + 1
        seg_kv = type(kv)(kv.k[:, a:].copy(), kv.v[:, a:].copy(), kv.positions[a:].copy())
        structural.append(T)
        toks += [np.array([0]), np.asarray(seg, np.int64)]
        target = np.arange(T + 1, T + 1 + len(seg), dtype=np.int64)
        hits.append(rounds.ToyHit(seg_kv, target))
        le.append((target, e))
        T += 1 + len(seg)
    label_entry = np.full(T, -1, np.int64)
    label_offset = np.full(T, -1, np.int64)
    for target, e in le:
        label_entry[target] = e
        label_offset[target] = np.arange(target.size)
    tokens = np.concatenate(toks)
    return rounds.ToyRequest(0, tokens, np.arange(T, dtype=np.int64),
                             np.arange(len(consumer_hist), dtype=np.int64),
                             np.asarray(structural, np.int64), hits, label_entry, label_offset)


def test_fidelity_brackets_with_recompute_fraction():
    """Acceptance C03 (test_acceptance.py:149-183) on the GPU: two outputs read
    in swapped order drift off their cached offsets; the mean K error against
    a full prefill is > 0 at r=0, non-increasing over r in {0, .15, .5, 1},
    and <= 1e-6 at r=1."""
    from paper_2604_03143_b200 import recompute, rounds
    w = rounds.toy_weights(4, 2, 8, 1024, seed=77)
    rng = np.random.default_rng(77)
    hist0, hist1 = rng.integers(1, 1024, 12), rng.integers(1, 1024, 14)
    out0, out1 = rng.integers(1, 1024, 10), rng.integers(1, 1024, 10)
    prep = _reuse_request(w, hist0, [(out1, hist1), (out0, hist0)])
    assert prep.hits[0].kv.positions[0] == 15 and prep.hits[1].kv.positions[0] == 13
    full = recompute.full_prefill(w, prep.tokens)
    errors = []
    for fraction in (0.0, 0.15, 0.5, 1.0):
        cfg = type("Cfg", (), {"recompute_fraction": fraction, "check_layer": 1})
        res = pic.recover_prepared(w, prep, cfg, CostLedger(4))
        dk = res.kv.k.cpu().numpy() - full.k
        errors.append(float(np.sqrt(np.einsum("lthd,lthd->lt", dk, dk)).mean()))
    assert errors[0] > 0.0
    assert all(b <= a for a, b in zip(errors, errors[1:])), errors
    assert errors[-1] <= 1e-6
