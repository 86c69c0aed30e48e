"""Pin the CPU oracle (oracle/roundkv_port.py) to the reference's own outputs.

Golden vectors were recorded by tests/golden/make_golden.py from roundkv
0.1.0 itself.  Integer/byte outputs (indices, slot maps, wire bytes) are
compared exactly everywhere; float digests are compared exactly on the
numpy build the goldens were recorded with (the trig bits come from numpy's
libm and are only guaranteed identical on the same build).
"""
import hashlib

import numpy as np
import pytest

from helpers import (violation_case, codec_trials, load_golden, load_npz, perturb, random_planes,
                     restore_trials, sha)
from oracle import roundkv_port as ref

G = load_golden()
SAME_NUMPY = G["numpy"] == np.__version__


def test_rope_digests_match_reference():
    for case in G["rope"]:
        rng = np.random.default_rng(case["seed"])
        t, h, d = case["shape"]
        k = rng.standard_normal((t, h, d)).astype(np.float32)
        pos = rng.integers(-8192, 8192, t).astype(np.int64)
        out = ref.rope_apply(k, pos, 10000.0)
        if SAME_NUMPY:
            assert sha(out) == case["sha"]
        # identities restated from pkg/tests/test_toymodel.py:62-80
        back = ref.rope_apply(out, -pos, 10000.0)
        assert np.abs(back - k).max() <= 1e-5


def test_rope_zero_delta_is_exact_copy():
    rng = np.random.default_rng(3)
    k = rng.standard_normal((12, 2, 8)).astype(np.float32)
    pos = np.arange(100, 112)
    out = ref.rope_recover(pos, pos, k)
    assert out is not k and np.array_equal(out, k)


def test_rope_validation():
    with pytest.raises(ValueError):
        ref.rope_apply(np.zeros((4, 2, 7), np.float32), np.arange(4))
    with pytest.raises(ValueError):
        ref.rope_apply(np.zeros((4, 2, 8), np.float32), np.arange(5))
    with pytest.raises(ValueError):
        ref.rope_apply(np.zeros((4, 8), np.float32), np.arange(4))


def _collector_jobs():
    meta = G["collector"]
    z = load_npz("collector.npz")
    jobs = []
    for a, agent in enumerate(meta["agents"]):
        for hit in agent["hits"]:
            m = hit["master"]
            jobs.append(ref.CollectJob(a, z[f"master{m}_k"], z[f"master{m}_v"],
                                       np.asarray(hit["target"], np.int64),
                                       np.asarray(hit["delta"], np.int64)))
    return meta, z, jobs


def test_collector_matches_reference_align_cached():
    meta, z, jobs = _collector_jobs()
    L, _, H, D = z["master0_k"].shape
    ctx = [(np.zeros((L, a["T"], H, D), np.float32), np.zeros((L, a["T"], H, D), np.float32))
           for a in meta["agents"]]
    calls = ref.collect_into_contexts(jobs, ctx, 10000.0)
    assert [1] * calls == meta["rope_calls_by_layer"]
    for a, agent in enumerate(meta["agents"]):
        shared = np.asarray(agent["shared_idx"])
        got_k = ctx[a][0][:, shared]
        want_k = z[f"agent{a}_k_shared"]
        assert np.abs(got_k - want_k).max() <= 1e-6
        if SAME_NUMPY:
            assert np.array_equal(got_k, want_k)
        assert np.array_equal(ctx[a][1][:, shared], z[f"agent{a}_v_shared"])


def test_collector_pool_form_equals_context_form():
    meta, z, jobs = _collector_jobs()
    L, _, H, D = z["master0_k"].shape
    ctx = [(np.zeros((L, a["T"], H, D), np.float32), np.zeros((L, a["T"], H, D), np.float32))
           for a in meta["agents"]]
    ref.collect_into_contexts(jobs, ctx, 10000.0)
    free = np.ones(512, bool)
    maps = [ref.allocate_slots(free, a["T"], 32) for a in meta["agents"]]
    pk = np.zeros((L, 512, H, D), np.float32)
    pv = np.zeros_like(pk)
    ref.collect_into_pool(jobs, maps, pk, pv, 10000.0)
    for a, agent in enumerate(meta["agents"]):
        shared = np.asarray(agent["shared_idx"])
        slots = maps[a][shared]
        assert np.array_equal(pk[:, slots], ctx[a][0][:, shared])
        assert np.array_equal(pv[:, slots], ctx[a][1][:, shared])


def test_codec_trials_match_reference():
    for trial, want in zip(codec_trials(len(G["codec_trials"])), G["codec_trials"]):
        layers = ref.encode_diff(trial.master_k, trial.master_v, trial.mirror_k,
                                 trial.mirror_v, trial.hints, trial.block_size)
        assert [ld.indices.tolist() for ld in layers] == want["indices"]
        L, T, H, D = trial.master_k.shape
        wire = ref.serialize(layers, trial.block_size, H, D, T)
        assert len(wire) == want["wire_len"]
        assert len(wire) == ref.wire_size([ld.indices.size for ld in layers],
                                          trial.block_size, H, D)
        assert hashlib.sha256(wire).hexdigest() == want["wire_sha"]
        _, back = ref.deserialize(wire)
        k, v = ref.decode_dense(trial.master_k, trial.master_v, back, trial.block_size)
        assert np.array_equal(k, trial.mirror_k) and np.array_equal(v, trial.mirror_v)


def test_known_answers():
    known = G["known"]
    rng = np.random.default_rng(known["worked"]["seed"])
    k, v, _ = random_planes(rng, 640)
    mk, mv, hints = perturb(rng, k, v, 32, [3, 17])
    layers = ref.encode_diff(k, v, mk, mv, hints, 32)
    payload = sum(ld.k_blocks.nbytes + ld.v_blocks.nbytes for ld in layers)
    assert payload == known["worked"]["payload"] == 32768
    wire = ref.serialize(layers, 32, 2, 8, 640)
    assert len(wire) - payload == 80
    assert hashlib.sha256(wire).hexdigest() == known["worked"]["wire_sha"]

    rng = np.random.default_rng(known["violation"]["seed"])
    k, v, _ = random_planes(rng, 128)
    mk, mv, hints = perturb(rng, k, v, 32, [1])
    mv[0, 100, 0, 0] += 0.5
    with pytest.raises(ref.HintViolation) as err:
        ref.encode_diff(k, v, mk, mv, hints, 32)
    assert str(err.value) == known["violation"]["message"]

    rng = np.random.default_rng(known["partial"]["seed"])
    k, v, _ = random_planes(rng, 70)
    mk, mv, hints = perturb(rng, k, v, 32, [2])
    layers = ref.encode_diff(k, v, mk, mv, hints, 32)
    assert np.all(layers[0].k_blocks[0, 6:] == 0.0)
    wire = ref.serialize(layers, 32, 2, 8, 70)
    assert hashlib.sha256(wire).hexdigest() == known["partial"]["wire_sha"]


def test_malformed_wire_rejected():
    rng = np.random.default_rng(41)
    k, v, _ = random_planes(rng, 64)
    mk, mv, hints = perturb(rng, k, v, 32, [0])
    wire = ref.serialize(ref.encode_diff(k, v, mk, mv, hints, 32), 32, 2, 8, 64)
    for bad, what in [(b"XXXX" + wire[4:], "magic"), (wire[:4] + b"\xff\x00" + wire[6:], "version"),
                      (wire[:10], "truncated"), (wire[:-6], "truncated"),
                      (wire + b"\x00", "trailing"), (b"", "truncated")]:
        with pytest.raises(ref.WireError, match=what):
            ref.deserialize(bad)
    flag = bytearray(wire)
    flag[28] = 7
    with pytest.raises(ref.WireError, match="flag"):
        ref.deserialize(bytes(flag))
    tail = bytearray(wire)
    tail[-4:] = (99).to_bytes(4, "little")
    with pytest.raises(ref.WireError, match="valid_len"):
        ref.deserialize(bytes(tail))


def test_restore_trials_match_reference():
    for trial, want in zip(restore_trials(len(G["restores"])), G["restores"]):
        layers = ref.encode_diff(trial.master_k, trial.master_v, trial.mirror_k,
                                 trial.mirror_v, trial.hints, trial.block_size)
        free = np.ones(128, bool)
        slots = ref.allocate_slots(free, trial.master_k.shape[1], 16)
        assert slots.tolist() == want["slots"]
        pk = np.zeros((3, 128, 2, 8), np.float32)
        pv = np.zeros_like(pk)
        new = trial.positions + trial.delta
        ref.fused_restore(trial.master_k, trial.master_v, layers, 16, trial.positions, new,
                          slots, pk, pv, 10000.0)
        if SAME_NUMPY:
            assert sha(pk[:, slots], pv[:, slots]) == want["sha"]
        dk = np.zeros_like(pk)
        dv = np.zeros_like(pk)
        ref.dense_restore(trial.master_k, trial.master_v, layers, 16, trial.positions, new,
                          slots, dk, dv, 10000.0)
        assert np.array_equal(pk, dk) and np.array_equal(pv, dv)


def test_family_matches_reference():
    fam = G["family"]
    z = load_npz("family.npz")
    bs = fam["block_size"]
    L, T, H, D = z["master_k"].shape
    for m in fam["mirrors"]:
        rid = m["rid"]
        layers = ref.encode_diff(z["master_k"], z["master_v"], z[f"mirror{rid}_k"],
                                 z[f"mirror{rid}_v"], z[f"hints{rid}"], bs)
        assert [ld.indices.tolist() for ld in layers] == m["indices"]
        wire = ref.serialize(layers, bs, H, D, T)
        assert hashlib.sha256(wire).hexdigest() == m["wire_sha"]
        slots = np.asarray(m["fused_slots"])
        cap = 4 * T + 32
        pk = np.zeros((L, cap, H, D), np.float32)
        pv = np.zeros_like(pk)
        pos = z["positions"]
        ref.fused_restore(z["master_k"], z["master_v"], layers, bs, pos, pos + 16, slots,
                          pk, pv, fam["rope_base"])
        if SAME_NUMPY:
            assert sha(pk[:, slots], pv[:, slots]) == m["fused_sha"]


def test_allocator_stream_matches_reference():
    free = np.ones(256, bool)
    live = {}
    for op in G["allocator"]:
        if op["op"] == "alloc":
            got = ref.allocate_slots(free, op["n"], 32)
            assert got.tolist() == op["slots"]
            live[op["serial"]] = got
        elif op["op"] == "free":
            free[live.pop(op["serial"])] = True


def test_selection_matches_reference_probe_and_select():
    sel = G["collector"]["selection"]
    z = load_npz("collector.npz")
    mags = ref.key_diff(z["sel_fresh"], z["sel_cached"])
    assert np.abs(mags - z["sel_mags"]).max() <= 1e-6
    off = 0
    devs = {}
    for m, n in enumerate(sel["counts"]):
        mm = mags[off:off + n]
        imp = ref.select_important(mm, ref.recompute_budget(sel["fraction"], n))
        assert imp.tolist() == sel["important_rel"][m]
        devs[m] = float(mm.sum())
        assert abs(devs[m] - sel["deviation"][m]) <= 1e-6 * max(1.0, abs(sel["deviation"][m]))
        off += n
    assert ref.select_master(devs) == sel["master"]


def test_toymodel_matches_reference():
    z = load_npz("toymodel.npz")
    for name, meta in G["toymodel"].items():
        L, H, D, V, seed = meta["config"]
        w = ref.build_weights(L, H, D, V, seed)
        assert sha(w.embed, w.wq, w.wk, w.wv, w.wm) == meta["weights_sha"]
        toks = z[f"{name}_tokens"]
        k, v = ref.full_prefill(w, toks)
        assert np.abs(k - z[f"{name}_prefill_k"]).max() <= 1e-6
        if SAME_NUMPY:
            assert sha(k, v) == meta["prefill_sha"]
        pos = np.arange(toks.size, dtype=np.int64) + 5
        k, v = ref.selective_forward(w, toks, pos, z[f"{name}_fix"], z[f"{name}_ctx_k"],
                                     z[f"{name}_ctx_v"])
        assert np.abs(k - z[f"{name}_sel_k"]).max() <= 1e-6
        assert np.abs(v - z[f"{name}_sel_v"]).max() <= 1e-6
        if SAME_NUMPY:
            assert sha(k, v) == meta["selective_sha"]


def test_selection_known_answers():
    fresh = np.zeros((3, 2, 4), np.float32)
    cached = np.zeros((3, 2, 4), np.float32)
    cached[1, 0, 0], cached[1, 1, 0] = 3.0, 4.0
    assert ref.key_diff(fresh, cached).tolist() == [0.0, 5.0, 0.0]
    mags = np.array([0.0, 3.0, 3.0, 1.0, 0.0, 2.0], np.float32)
    assert ref.select_important(mags, 3).tolist() == [1, 2, 5]
    assert ref.select_important(mags, 10).tolist() == [1, 2, 3, 5]
    assert ref.select_important(mags, 0).tolist() == []
    assert ref.select_important(np.array([5.0, 5.0, 5.0, 1.0], np.float32), 2).tolist() == [0, 1]


def test_select_master_and_budget():
    assert ref.select_master({0: 2.0, 1: 1.5, 2: 3.0}) == 1
    assert ref.select_master({2: 1.5, 0: 1.5, 1: 2.0}) == 0
    assert ref.recompute_budget(0.15, 20) == 3
    assert ref.recompute_budget(0.15, 21) == 4


def test_segment_index_port_matches_reference_stream():
    from helpers import replay_segment_index

    class E:
        _n = 0

        def __init__(self, tok, nbytes, kv_ref):
            import hashlib
            self.digest = hashlib.blake2b(np.asarray([tok], dtype="<u4").tobytes(),
                                          digest_size=16).digest()
            self.nbytes, self.kv_ref = nbytes, kv_ref
            E._n += 1
            self.entry_id = E._n

    replay_segment_index(lambda b, p, ev: ref.SegmentIndexPort(b, p, ev), E, G["segment_index"])


def test_oracle_violation_magnitudes_with_nan_inf_and_signed_zero():
    """NaN / inf / -0.0 outside the hints: the oracle's soundness message is
    the reference's, byte for byte (golden.json known.violation_special)."""
    for entry in G["known"]["violation_special"]:
        k, v, mk, mv, hints = violation_case(entry["case"])
        if entry["message"] is None:
            ref.encode_diff(k, v, mk, mv, hints, 32)
            continue
        with pytest.raises(ref.HintViolation) as err:
            ref.encode_diff(k, v, mk, mv, hints, 32)
        assert str(err.value) == entry["message"], entry["case"]


def test_product_value_types_match_the_reference():
    """ModelConfig / build_weights / PicConfig / ReuseGroup are the reference's
    (toymodel.py:36-57, core.py:38-66, pic.py:36-48, collective.py:40-59):
    weights bit-identical to the oracle's pinned restatement, same validation."""
    import paper_2604_03143_b200 as tk
    cfg = tk.ModelConfig(num_layers=3, num_heads=2, head_dim=8, vocab_size=64, weight_seed=7)
    assert cfg.hidden_dim == 16 and cfg.separator_token == 63
    w = tk.build_weights(cfg)
    o = ref.build_weights(3, 2, 8, 64, 7)
    for name in ("embed", "wq", "wk", "wv", "wm"):
        assert np.array_equal(getattr(w, name), getattr(o, name)), name
    for bad in (dict(head_dim=7), dict(num_layers=0), dict(vocab_size=1), dict(rope_base=0.0)):
        with pytest.raises(ValueError):
            tk.ModelConfig(**bad)
    assert tk.PicConfig().recompute_fraction == 0.15 and tk.PicConfig().check_layer == 1
    for bad in (dict(recompute_fraction=1.5), dict(check_layer=-1)):
        with pytest.raises(ValueError):
            tk.PicConfig(**bad)

    class _M:
        def __init__(self, rid):
            self.request_id = rid
    g = tk.ReuseGroup(3, [_M(1), _M(4)])
    assert g.member_ids == [1, 4] and len(g) == 2
    with pytest.raises(ValueError):
        tk.ReuseGroup(0, [_M(1)])
    with pytest.raises(ValueError):
        tk.ReuseGroup(0, [_M(1), _M(1)])


def test_oracle_neox_rotation_is_rotate_half():
    """oracle.rope_apply_neox (the collector's rope_style="neox" checker)
    equals the usual rotate-half formula q*cos + rotate_half(q)*sin with the
    reference's angles, and reduces to rope_apply on a head whose halves are
    the interleaved pairs."""
    rng = np.random.default_rng(0)
    k = rng.standard_normal((5, 3, 16)).astype(np.float32)
    pos = np.array([0, 3, 17, -4, 900])
    th = pos[:, None] * ref.inv_freq(16)[None, :]
    cos = np.concatenate([np.cos(th)] * 2, axis=-1)[:, None, :]
    sin = np.concatenate([np.sin(th)] * 2, axis=-1)[:, None, :]
    x = k.astype(np.float64)
    rot_half = np.concatenate([-x[..., 8:], x[..., :8]], axis=-1)
    assert np.array_equal(ref.rope_apply_neox(k, pos), (x * cos + rot_half * sin).astype(np.float32))
    # a permutation maps one pairing onto the other
    perm = np.stack([np.arange(8), np.arange(8, 16)], axis=-1).reshape(-1)   # (j, j + 8) -> (2j, 2j+1)
    assert np.array_equal(ref.rope_apply_neox(k, pos)[..., perm], ref.rope_apply(k[..., perm], pos))
