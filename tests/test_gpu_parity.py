"""GPU parity: every kernel through the C-ABI against the CPU oracle and the
reference's golden vectors.

Tolerances (north_star): float32 rotated keys / reconstructed KV max-abs
1e-5 (the fp64 rotation is expected to be bit-exact whenever the device's
cos/sin bits equal numpy's); bf16 within 1e-2 * max(1, |ref|) against the
oracle run on the f32-upcast inputs (one bf16 rounding of the output alone
is 2^-9 relative); V rows, diff masks, block indices, payload layout, slot
maps and wire bytes are bit-exact.
"""
import hashlib

import numpy as np
import pytest
import torch

import paper_2604_03143_b200 as tk
from helpers import (violation_case, codec_trials, load_golden, load_npz, perturb, random_planes,
                     restore_trials, sha)
from oracle import roundkv_port as ref
from paper_2604_03143_b200 import rounds

pytestmark = pytest.mark.gpu
G = load_golden()
DEV = torch.device("cuda", 0)
F32_TOL = 1e-5


def bf16_close(got: np.ndarray, want: np.ndarray) -> float:
    """max |got - want| / max(1, |want|)"""
    return float((np.abs(got - want) / np.maximum(1.0, np.abs(want))).max()) if got.size else 0.0


@pytest.fixture(scope="module", autouse=True)
def _built():
    tk.build_library()
    assert torch.cuda.is_available()


# ---------------------------------------------------------------------------
# rotary


def test_rope_apply_matches_oracle_and_reference_digests():
    exact = 0
    for case in G["rope"]:
        rng = np.random.default_rng(case["seed"])
        t, h, d = case["shape"]
        k = rng.standard_normal((t, h, d)).astype(np.float32)
        pos = rng.integers(-8192, 8192, t).astype(np.int64)
        got = tk.rope_apply(k, pos)
        want = ref.rope_apply(k, pos)
        assert isinstance(got, np.ndarray) and got.dtype == np.float32
        assert np.abs(got - want).max() <= F32_TOL
        exact += int(np.array_equal(got, want))
    print(f"rope cases bit-exact with numpy: {exact}/{len(G['rope'])}")


def test_rope_identities_on_device():
    rng = np.random.default_rng(5)
    k = torch.from_numpy((rng.standard_normal((20, 2, 8)) * 0.05).astype(np.float32)).to(DEV)
    p = np.arange(100, 120, dtype=np.int64)
    q = np.arange(20, dtype=np.int64) * 3 + 1
    a = tk.rope_apply(tk.rope_apply(k, p), q)
    b = tk.rope_apply(k, p + q)
    assert (a - b).abs().max().item() <= 1e-6
    assert (tk.rope_apply(tk.rope_apply(k, p), -p) - k).abs().max().item() <= 1e-6
    span = tk.PositionSpan.identity(range(100, 120))
    out = tk.rope_recover(span, k)
    assert out is not k and torch.equal(out, k)
    with pytest.raises(ValueError):
        tk.rope_apply(np.zeros((4, 2, 7), np.float32), np.arange(4))
    with pytest.raises(ValueError):
        tk.rope_apply(np.zeros((4, 2, 8), np.float32), np.arange(5))


def test_rope_bf16_close_to_oracle():
    rng = np.random.default_rng(8)
    k = rng.standard_normal((64, 4, 128)).astype(np.float32)
    pos = rng.integers(-8192, 8192, 64)
    kb = torch.from_numpy(k).to(DEV).bfloat16()
    got = tk.rope_apply(kb, pos).float().cpu().numpy()
    want = ref.rope_apply(kb.float().cpu().numpy(), pos)
    assert bf16_close(got, want) <= 1e-2


# ---------------------------------------------------------------------------
# collector


class _Hit:
    def __init__(self, kv, target, delta):
        self.kv = kv
        self.target_idx = np.asarray(target, np.int64)
        self.delta = np.asarray(delta, np.int64)


class _Member:
    def __init__(self, hits):
        self.hits = hits


def _golden_round():
    meta = G["collector"]
    z = load_npz("collector.npz")
    masters = [tk.LayeredKv(z[f"master{i}_k"], z[f"master{i}_v"], z[f"master{i}_pos"])
               for i in range(len(meta["agents"]))]
    members = [_Member([_Hit(masters[h["master"]], h["target"], h["delta"]) for h in a["hits"]])
               for a in meta["agents"]]
    return meta, z, masters, members


def test_align_cached_dropin_matches_reference_goldens():
    meta, z, masters, members = _golden_round()
    L, _, H, D = z["master0_k"].shape
    ctx = [(np.zeros((L, a["T"], H, D), np.float32), np.zeros((L, a["T"], H, D), np.float32))
           for a in meta["agents"]]
    ledger = tk.CostLedger(L)
    tk.skeleton_values(members, ctx)
    tk.align_cached(members, ctx, 10000.0, ledger)
    assert ledger.rope_calls_by_layer == meta["rope_calls_by_layer"]
    for a, agent in enumerate(meta["agents"]):
        shared = np.asarray(agent["shared_idx"])
        assert np.abs(ctx[a][0][:, shared] - z[f"agent{a}_k_shared"]).max() <= 1e-6
        assert np.array_equal(ctx[a][1][:, shared], z[f"agent{a}_v_shared"])
        others = np.setdiff1d(np.arange(agent["T"]), shared)
        assert not ctx[a][0][:, others].any() and not ctx[a][1][:, others].any()


def test_align_cached_device_contexts():
    meta, z, masters, members = _golden_round()
    L, _, H, D = z["master0_k"].shape
    dev_masters = [tk.LayeredKv(torch.from_numpy(m.k).to(DEV), torch.from_numpy(m.v).to(DEV),
                                m.positions) for m in masters]
    members = [_Member([_Hit(dev_masters[masters.index(h.kv)], h.target_idx, h.delta)
                        for h in m.hits]) for m in members]
    ctx = [(torch.zeros((L, a["T"], H, D), device=DEV), torch.zeros((L, a["T"], H, D), device=DEV))
           for a in meta["agents"]]
    tk.align_cached(members, ctx, 10000.0)
    tk.skeleton_values(members, ctx)
    for a, agent in enumerate(meta["agents"]):
        shared = np.asarray(agent["shared_idx"])
        k = ctx[a][0].cpu().numpy()
        assert np.abs(k[:, shared] - z[f"agent{a}_k_shared"]).max() <= 1e-6
        assert np.array_equal(ctx[a][1].cpu().numpy()[:, shared], z[f"agent{a}_v_shared"])


def test_align_cached_host_contexts_chunked_readback():
    """configs[0]-sized host contexts take the chunked, threaded read-back
    (one chunk per member run): equal to the oracle collector (V bit for bit,
    K bit for bit in float32); a member whose hits overlap keeps the serial
    last-write-wins result; two members sharing one context fall back to one
    chunk and still match a serial scatter."""
    spec = rounds.CONFIGS["c1"]
    mk, mv = rounds.master_planes_host(spec)
    src = rounds.source_offsets(spec)
    L, H, D, n = spec.num_layers, spec.num_heads, spec.head_dim, spec.seg_len
    masters = [tk.LayeredKv(np.ascontiguousarray(mk[:, g * n:(g + 1) * n]),
                            np.ascontiguousarray(mv[:, g * n:(g + 1) * n]),
                            np.arange(src[g], src[g] + n)) for g in range(spec.total_segments)]
    T = spec.tokens_per_agent
    members, jobs = [], []
    for a in range(spec.num_agents):
        starts = rounds.segment_starts(spec, a)
        hits = []
        for sgm in range(spec.num_segments):
            tgt = np.arange(starts[sgm], starts[sgm] + n, dtype=np.int64)
            hits.append(_Hit(masters[sgm], tgt, tgt - masters[sgm].positions))
        if a == 3:      # a late hit overwriting part of an earlier one
            part = tk.LayeredKv(np.ascontiguousarray(masters[1].k[:, :n // 2]),
                                np.ascontiguousarray(masters[1].v[:, :n // 2]),
                                masters[1].positions[:n // 2])
            tgt = np.arange(starts[0] + 5, starts[0] + 5 + n // 2, dtype=np.int64)
            hits.append(_Hit(part, tgt, tgt - part.positions))
        for h in hits:
            jobs.append(ref.CollectJob(a, h.kv.k, h.kv.v, h.target_idx, h.delta))
        members.append(_Member(hits))
    ctx = [(np.zeros((L, T, H, D), np.float32), np.zeros((L, T, H, D), np.float32))
           for _ in range(spec.num_agents)]
    want = [(np.zeros((L, T, H, D), np.float32), np.zeros((L, T, H, D), np.float32))
            for _ in range(spec.num_agents)]
    tk.skeleton_values(members, ctx)
    tk.align_cached(members, ctx, 10000.0)
    ref.collect_into_contexts(jobs, want, 10000.0)
    for a in range(spec.num_agents):
        assert np.array_equal(ctx[a][1], want[a][1])
        assert np.array_equal(ctx[a][0], want[a][0])
    # members 0 and 1 share one context pair: serial order, member 1 last
    shared = (np.zeros((L, T, H, D), np.float32), np.zeros((L, T, H, D), np.float32))
    ctx2 = [shared, shared] + ctx[2:]
    tk.align_cached(members, ctx2, 10000.0)
    want2 = (np.zeros((L, T, H, D), np.float32), np.zeros((L, T, H, D), np.float32))
    ref.collect_into_contexts([j for j in jobs if j.agent in (0, 1)],
                              [want2, want2], 10000.0)
    assert np.array_equal(shared[0], want2[0])


def _collect_case(spec: rounds.RoundSpec, tile_rows=None, seed=0):
    """Run the pool-form collector on a synthetic round and the oracle on the
    same (f32-upcast) inputs; return (pool_k, pool_v, want_k, want_v, slots)."""
    mk, mv = rounds.master_planes_host(spec, seed)
    dt = spec.torch_dtype
    arena_k = torch.from_numpy(mk).to(DEV).to(dt)
    arena_v = torch.from_numpy(mv).to(DEV).to(dt)
    arena = rounds.make_arena(spec, arena_k, arena_v)
    T = spec.tokens_per_agent
    pool = tk.PagedPool(spec.num_agents * T + 64, spec.num_layers, spec.num_heads, spec.head_dim,
                        dtype=dt, device=DEV)
    maps = [pool.allocate(T, a) for a in range(spec.num_agents)]
    jobs = [j for a in range(spec.num_agents) for j in rounds.agent_jobs(spec, a, maps[a].slots)]
    col = tk.KVCollector(arena, pool, 10000.0, tile_rows=tile_rows)
    plan = col.plan(jobs)
    ledger = tk.CostLedger(spec.num_layers)
    col.collect(plan, ledger)
    assert ledger.rope_calls_by_layer == [1] * spec.num_layers
    # oracle on the upcast inputs
    mk32 = arena_k.float().cpu().numpy()
    mv32 = arena_v.float().cpu().numpy()
    cap = pool.capacity
    want_k = np.zeros((spec.num_layers, cap, spec.num_heads, spec.head_dim), np.float32)
    want_v = np.zeros_like(want_k)
    ojobs = []
    for j in jobs:
        r0 = j.segment * spec.seg_len
        ojobs.append(ref.CollectJob(0, mk32[:, r0:r0 + spec.seg_len], mv32[:, r0:r0 + spec.seg_len],
                                    np.arange(spec.seg_len), j.delta))
    # each oracle job writes its own destination rows
    for j, oj in zip(jobs, ojobs):
        ref.collect_into_pool([oj], [j.dst_rows], want_k, want_v, 10000.0)
    return pool.k.float().cpu().numpy(), pool.v.float().cpu().numpy(), want_k, want_v, jobs


def test_collector_c1_f32_matches_oracle():
    spec = rounds.CONFIGS["c1"]
    gk, gv, wk, wv, jobs = _collect_case(spec)
    rows = np.concatenate([j.dst_rows for j in jobs])
    assert np.array_equal(gv[:, rows], wv[:, rows])
    err = np.abs(gk[:, rows] - wk[:, rows]).max()
    exact = float(np.mean(gk[:, rows] == wk[:, rows]))
    print(f"c1 collector max-abs {err:.3e}, bit-exact fraction {exact:.8f}")
    assert err <= F32_TOL
    untouched = np.setdiff1d(np.arange(gk.shape[1]), rows)
    assert not gk[:, untouched].any() and not gv[:, untouched].any()


@pytest.mark.parametrize("tile_rows", [None, 1, 7])
def test_collector_bf16_reduced_c2(tile_rows):
    spec = rounds.CONFIGS["c2"].scaled(num_layers=3, num_agents=6, num_segments=5, hist_len=40)
    gk, gv, wk, wv, jobs = _collect_case(spec, tile_rows=tile_rows)
    rows = np.concatenate([j.dst_rows for j in jobs])
    assert np.array_equal(gv[:, rows], wv[:, rows])
    assert bf16_close(gk[:, rows], wk[:, rows]) <= 1e-2


def test_collector_multi_session_c3_shape():
    spec = rounds.CONFIGS["c3"].scaled(num_layers=2, num_agents=12, sessions=3, hist_len=17)
    gk, gv, wk, wv, jobs = _collect_case(spec)
    rows = np.concatenate([j.dst_rows for j in jobs])
    assert {j.segment for j in jobs} == set(range(spec.total_segments))
    assert np.array_equal(gv[:, rows], wv[:, rows])
    assert bf16_close(gk[:, rows], wk[:, rows]) <= 1e-2


def test_collector_odd_shapes_and_chunking():
    # rows that are not 16-byte multiples (pair-unit path, no bulk copy),
    # many agents over few tiles (job chunking)
    for spec in [rounds.RoundSpec("odd", 2, 3, 6, "f32", 40, 2, 5, 3),
                 rounds.RoundSpec("odd16", 1, 1, 2, "bf16", 30, 3, 9, 1),
                 rounds.RoundSpec("many", 1, 2, 8, "f32", 300, 1, 3, 2)]:
        gk, gv, wk, wv, jobs = _collect_case(spec)
        rows = np.concatenate([j.dst_rows for j in jobs])
        assert np.array_equal(gv[:, rows], wv[:, rows])
        if spec.dtype == "f32":
            assert np.abs(gk[:, rows] - wk[:, rows]).max() <= F32_TOL
        else:
            assert bf16_close(gk[:, rows], wk[:, rows]) <= 1e-2


def test_collector_per_token_and_zero_deltas():
    rng = np.random.default_rng(12)
    L, H, D, n = 2, 2, 16, 37
    mk = rng.standard_normal((L, n, H, D)).astype(np.float32)
    mv = rng.standard_normal((L, n, H, D)).astype(np.float32)
    arena = tk.MasterArena(torch.from_numpy(mk).to(DEV), torch.from_numpy(mv).to(DEV),
                           [0], [n], [np.arange(n)])
    pool = tk.PagedPool(256, L, H, D, device=DEV)
    m0, m1 = pool.allocate(n), pool.allocate(n)
    d_var = rng.integers(-5000, 5000, n).astype(np.int64)
    for deltas in ([np.zeros(n, np.int64), np.zeros(n, np.int64)],
                   [d_var, np.full(n, 17, np.int64)]):
        jobs = [tk.CollectJob(0, m0.slots, deltas[0]), tk.CollectJob(0, m1.slots, deltas[1])]
        col = tk.KVCollector(arena, pool)
        col.collect(col.plan(jobs))
        gk = pool.k.cpu().numpy()
        for m, d in zip((m0, m1), deltas):
            for layer in range(L):
                want = ref.rope_recover(np.zeros(n), d, mk[layer]) if d.any() else mk[layer]
                assert np.abs(gk[layer, m.slots] - want).max() <= F32_TOL
                if not d.any():
                    assert np.array_equal(gk[layer, m.slots], mk[layer])


# ---------------------------------------------------------------------------
# encoder / decoder


def test_codec_trials_match_reference_goldens():
    for trial, want in zip(codec_trials(len(G["codec_trials"])), G["codec_trials"]):
        master = tk.LayeredKv(trial.master_k, trial.master_v, trial.positions)
        mirror = tk.LayeredKv(trial.mirror_k, trial.mirror_v, trial.positions)
        blocks = tk.CacheBlockConfig(trial.block_size)
        diff = tk.encode_diff(master, mirror, trial.hints, blocks)
        assert [ld.indices.tolist() for ld in diff.layers] == want["indices"]
        wire = tk.serialize_diff(diff)
        assert len(wire) == want["wire_len"] == tk.wire_nbytes(diff)
        assert hashlib.sha256(wire).hexdigest() == want["wire_sha"]
        back = tk.diff_decode_dense(master, tk.deserialize_diff(wire))
        assert np.array_equal(back.k, trial.mirror_k) and np.array_equal(back.v, trial.mirror_v)
        direct = tk.diff_decode_dense(master, diff)
        assert np.array_equal(direct.k, trial.mirror_k)


def test_known_answers_and_errors():
    known = G["known"]
    blocks = tk.CacheBlockConfig(32)
    rng = np.random.default_rng(known["worked"]["seed"])
    k, v, pos = random_planes(rng, 640)
    mk, mv, hints = perturb(rng, k, v, 32, [3, 17])
    diff = tk.encode_diff(tk.LayeredKv(k, v, pos), tk.LayeredKv(mk, mv, pos), hints, blocks)
    assert diff.changed_blocks_per_layer == [2, 2, 2, 2]
    assert diff.payload_nbytes == 32768
    wire = tk.serialize_diff(diff)
    assert len(wire) - diff.payload_nbytes == 80
    assert hashlib.sha256(wire).hexdigest() == known["worked"]["wire_sha"]

    rng = np.random.default_rng(known["violation"]["seed"])
    k, v, pos = random_planes(rng, 128)
    mk, mv, hints = perturb(rng, k, v, 32, [1])
    mv[0, 100, 0, 0] += 0.5
    with pytest.raises(tk.HintSoundnessError) as err:
        tk.encode_diff(tk.LayeredKv(k, v, pos), tk.LayeredKv(mk, mv, pos), hints, blocks)
    assert str(err.value) == known["violation"]["message"]

    rng = np.random.default_rng(known["partial"]["seed"])
    k, v, pos = random_planes(rng, 70)
    mk, mv, hints = perturb(rng, k, v, 32, [2])
    diff = tk.encode_diff(tk.LayeredKv(k, v, pos), tk.LayeredKv(mk, mv, pos), hints, blocks)
    assert diff.layers[0].k_blocks.shape[1] == 32
    assert np.all(diff.layers[0].k_blocks[0, 6:] == 0.0)
    assert hashlib.sha256(tk.serialize_diff(diff)).hexdigest() == known["partial"]["wire_sha"]

    with pytest.raises(ValueError, match="shape"):
        tk.encode_diff(tk.LayeredKv(k, v, pos), tk.LayeredKv(*random_planes(rng, 96)[:2],
                                                             np.arange(96)), hints, blocks)
    k2, v2, _ = random_planes(rng, 70)
    with pytest.raises(ValueError, match="positions"):
        tk.encode_diff(tk.LayeredKv(k, v, pos), tk.LayeredKv(k2, v2, pos + 5), hints, blocks)


def test_violation_magnitudes_with_nan_inf_and_signed_zero():
    """K2's soundness error for NaN / inf / -0.0 outside the hints equals the
    reference's message byte for byte: numpy's per-plane max propagates NaN,
    Python's max(k, v) keeps K's NaN and drops V's (diffstore.py:157-160)."""
    blocks = tk.CacheBlockConfig(32)
    for entry in G["known"]["violation_special"]:
        k, v, mk, mv, hints = violation_case(entry["case"])
        pos = np.arange(k.shape[1])
        for dev in (False, True):
            conv = (lambda a: torch.from_numpy(a).to(DEV)) if dev else (lambda a: a)
            master = tk.LayeredKv(conv(k), conv(v), pos)
            mirror = tk.LayeredKv(conv(mk), conv(mv), pos)
            if entry["message"] is None:
                tk.encode_diff(master, mirror, hints, blocks)
                continue
            with pytest.raises(tk.HintSoundnessError) as err:
                tk.encode_diff(master, mirror, hints, blocks)
            assert str(err.value) == entry["message"], (entry["case"], dev)


def test_float_equality_semantics():
    """+0 == -0 is unchanged, NaN != NaN is changed (np.array_equal)."""
    k = np.zeros((1, 64, 1, 4), np.float32)
    v = np.zeros_like(k)
    pos = np.arange(64)
    mk = k.copy()
    mk[0, 3, 0, 0] = -0.0
    d = tk.encode_diff(tk.LayeredKv(k, v, pos), tk.LayeredKv(mk, v.copy(), pos),
                       np.empty(0, np.int64), tk.CacheBlockConfig(32))
    assert d.changed_blocks_per_layer == [0]
    k2 = k.copy()
    k2[0, 40, 0, 1] = np.nan
    d = tk.encode_diff(tk.LayeredKv(k2, v, pos), tk.LayeredKv(k2.copy(), v.copy(), pos),
                       np.arange(32, 64), tk.CacheBlockConfig(32))
    assert d.layers[0].indices.tolist() == [1]


def test_hinted_but_identical_not_stored_and_single_row_change():
    rng = np.random.default_rng(23)
    k, v, pos = random_planes(rng, 128)
    mk, mv, _ = perturb(rng, k, v, 32, [1])
    d = tk.encode_diff(tk.LayeredKv(k, v, pos), tk.LayeredKv(mk, mv, pos), np.arange(128),
                       tk.CacheBlockConfig(32))
    assert d.changed_blocks_per_layer == [1, 1, 1, 1]
    m2 = k.copy()
    m2[2, 40, 1, 3] += 1.0
    d = tk.encode_diff(tk.LayeredKv(k, v, pos), tk.LayeredKv(m2, v.copy(), pos), np.array([40]),
                       tk.CacheBlockConfig(32))
    assert d.changed_blocks_per_layer == [0, 0, 1, 0] and d.layers[2].indices.tolist() == [1]


def test_family_matches_reference_stats():
    fam = G["family"]
    z = load_npz("family.npz")
    pos = z["positions"]
    results = {fam["master_id"]: type("R", (), {"kv": tk.LayeredKv(z["master_k"], z["master_v"], pos)})}
    hints = {}
    for m in fam["mirrors"]:
        rid = m["rid"]
        results[rid] = type("R", (), {"kv": tk.LayeredKv(z[f"mirror{rid}_k"], z[f"mirror{rid}_v"], pos)})
        hints[rid] = z[f"hints{rid}"]
    plan = type("P", (), {"master_id": fam["master_id"], "mirror_diff_hints": hints})
    store = tk.DiffStore(tk.CacheBlockConfig(fam["block_size"]))
    enc = store.encode_family(plan, results)
    st = fam["stats"]
    assert enc.stats.dense_nbytes == st["dense"]
    assert enc.stats.diff_payload_nbytes == st["payload"]
    assert enc.stats.diff_serialized_nbytes == st["serialized"]
    assert enc.stats.changed_blocks == st["changed"]
    assert enc.stats.ratios == st["ratios"]
    assert enc.stats.family_cost == st["family_cost"]
    assert enc.master.pin_count == len(fam["mirrors"])
    L, T, H, D = z["master_k"].shape
    for m in fam["mirrors"]:
        h = enc.mirrors[m["rid"]]
        assert [ld.indices.tolist() for ld in h.diff.layers] == m["indices"]
        assert hashlib.sha256(tk.serialize_diff(h.diff)).hexdigest() == m["wire_sha"]
        pool = tk.PagedPool(4 * T + 32, L, H, D, block_size=8, device=DEV)
        fmap = pool.allocate(T, 1)
        dmap = pool.allocate(T, 2)
        assert fmap.slots.tolist() == m["fused_slots"]
        span = tk.PositionSpan.shifted(pos, 16)
        led = tk.CostLedger(L)
        tk.fused_restore(h, span, pool, fmap, fam["rope_base"], ledger=led)
        tk.dense_restore(h, span, pool, dmap, fam["rope_base"])
        assert led.bytes_moved == m["bytes_moved"] and led.temp_buffer_peak_bytes == m["temp_peak"]
        fk = np.stack([pool.read_rows(fmap, l, host=True)[0] for l in range(L)])
        dk = np.stack([pool.read_rows(dmap, l, host=True)[0] for l in range(L)])
        assert np.array_equal(fk, dk)
    for h in enc.mirrors.values():
        h.release()
    store.drop_family(enc.master.family_id)


# ---------------------------------------------------------------------------
# restores


def _handle(master_k, master_v, pos, diff):
    master = tk.MasterEntry(0, tk.LayeredKv(master_k, master_v, pos))
    master.pin_count = 1
    return tk.MirrorHandle(0, 1, master, diff)


def test_restore_trials_match_oracle_and_goldens():
    exact = 0
    for trial, want in zip(restore_trials(len(G["restores"])), G["restores"]):
        master = tk.LayeredKv(trial.master_k, trial.master_v, trial.positions)
        mirror = tk.LayeredKv(trial.mirror_k, trial.mirror_v, trial.positions)
        diff = tk.encode_diff(master, mirror, trial.hints, tk.CacheBlockConfig(16))
        handle = _handle(trial.master_k, trial.master_v, trial.positions, diff)
        span = tk.PositionSpan.shifted(trial.positions, trial.delta)
        pool = tk.PagedPool(128, 3, 2, 8, block_size=16, device=DEV)
        smap = pool.allocate(trial.master_k.shape[1], 1)
        assert smap.slots.tolist() == want["slots"]
        led = tk.CostLedger(3)
        tk.fused_restore(handle, span, pool, smap, 10000.0, ledger=led)
        assert led.bytes_moved == want["bytes_moved"]
        gk = np.stack([pool.read_rows(smap, l, host=True)[0] for l in range(3)])
        gv = np.stack([pool.read_rows(smap, l, host=True)[1] for l in range(3)])
        layers = ref.encode_diff(trial.master_k, trial.master_v, trial.mirror_k, trial.mirror_v,
                                 trial.hints, 16)
        wk = np.zeros((3, 128, 2, 8), np.float32)
        wv = np.zeros_like(wk)
        ref.fused_restore(trial.master_k, trial.master_v, layers, 16, trial.positions,
                          trial.positions + trial.delta, smap.slots, wk, wv, 10000.0)
        assert np.array_equal(gv, wv[:, smap.slots])
        assert np.abs(gk - wk[:, smap.slots]).max() <= F32_TOL
        exact += int(sha(gk, gv) == want["sha"])
    print(f"restores bit-identical to the reference digests: {exact}/{len(G['restores'])}")


@pytest.mark.parametrize("offset", [0, 16, -5])
def test_fused_equals_dense_bitwise(offset):
    rng = np.random.default_rng(101 + offset)
    for _ in range(10):
        T = int(rng.integers(33, 161))
        nb = -(-T // 32)
        picks = sorted(rng.choice(nb, size=int(rng.integers(1, nb + 1)), replace=False).tolist())
        k, v, pos = random_planes(rng, T, start=int(rng.integers(0, 50)))
        mk, mv, hints = perturb(rng, k, v, 32, picks)
        diff = tk.encode_diff(tk.LayeredKv(k, v, pos), tk.LayeredKv(mk, mv, pos), hints,
                              tk.CacheBlockConfig(32))
        h = _handle(k, v, pos, diff)
        span = tk.PositionSpan.shifted(pos, offset)
        pool = tk.PagedPool(512, 4, 2, 8, device=DEV)
        a, b = pool.allocate(T, 1), pool.allocate(T, 2)
        tk.fused_restore(h, span, pool, a, 10000.0)
        tk.dense_restore(h, span, pool, b, 10000.0)
        for layer in range(4):
            fa = pool.read_rows(a, layer, host=True)
            fb = pool.read_rows(b, layer, host=True)
            assert np.array_equal(fa[0], fb[0]) and np.array_equal(fa[1], fb[1])
        if offset == 0:
            assert np.array_equal(np.stack([pool.read_rows(a, l, host=True)[0] for l in range(4)]), mk)


def test_restore_event_order_accounting_and_validation():
    rng = np.random.default_rng(17)
    k, v, pos = random_planes(rng, 96)
    mk, mv, hints = perturb(rng, k, v, 32, [0, 2])
    diff = tk.encode_diff(tk.LayeredKv(k, v, pos), tk.LayeredKv(mk, mv, pos), hints,
                          tk.CacheBlockConfig(32))
    h = _handle(k, v, pos, diff)
    pool = tk.PagedPool(512, 4, 2, 8, device=DEV)
    span = tk.PositionSpan.shifted(pos, 4)
    trace = []
    fl = tk.CostLedger(4)
    tk.fused_restore(h, span, pool, pool.allocate(96, 1), 10000.0, ledger=fl, trace=trace)
    assert trace == [(e, l) for l in range(4) for e in ("load", "swap", "diff", "rope", "write")]
    pair = 2 * 96 * 2 * 8 * 4
    assert fl.bytes_moved == 2 * 4 * 96 * 2 * 8 * 4 + diff.payload_nbytes
    assert fl.temp_buffer_peak_bytes == 2 * pair and fl.dense_mirror_allocations == 0
    dl = tk.CostLedger(4)
    dtrace = []
    tk.dense_restore(h, span, pool, pool.allocate(96, 2), 10000.0, ledger=dl, trace=dtrace)
    assert dtrace[0] == ("materialize", -1)
    assert dl.dense_mirror_allocations == 1 and dl.temp_buffer_peak_bytes == 4 * pair
    with pytest.raises(ValueError, match="one slot per token"):
        tk.fused_restore(h, span, pool, pool.allocate(32, 3), 10000.0)
    with pytest.raises(ValueError, match="source positions"):
        tk.fused_restore(h, tk.PositionSpan.shifted(pos + 3, 1), pool, pool.allocate(96, 4), 1e4)
    h.release()
    with pytest.raises(ValueError, match="released"):
        tk.fused_restore(h, span, pool, pool.allocate(96, 5), 10000.0)


# ---------------------------------------------------------------------------
# pool


def test_pool_roundtrip_poison_and_use_after_free():
    pool = tk.PagedPool(128, 3, 2, 8, device=DEV)
    rng = np.random.default_rng(0)
    m = pool.allocate(40, 1)
    assert m.slots.tolist() == list(range(40))
    stored = []
    for layer in range(3):
        kr = rng.standard_normal((40, 2, 8)).astype(np.float32)
        vr = rng.standard_normal((40, 2, 8)).astype(np.float32)
        pool.write_rows(m, layer, kr, vr)
        stored.append((kr, vr))
    for layer in range(3):
        kr, vr = pool.read_rows(m, layer, host=True)
        assert np.array_equal(kr, stored[layer][0]) and np.array_equal(vr, stored[layer][1])
    pool.free(m)
    assert torch.isnan(pool.k[:, :40]).all()
    with pytest.raises(tk.UseAfterFreeError):
        pool.read_rows(m, 0)
    m2 = pool.allocate(8)
    with pytest.raises(tk.UseAfterFreeError):
        pool.read_rows(m2, 0)
    with pytest.raises(tk.OutOfSlotsError):
        pool.allocate(500)


# ---------------------------------------------------------------------------
# full-size properties (BASELINE configs), size-independent checks


def test_c2_full_size_collector_and_codec_properties():
    spec = rounds.CONFIGS["c2"].scaled(num_agents=8)
    mk, mv = rounds.master_planes_host(spec)
    dt = spec.torch_dtype
    arena = rounds.make_arena(spec, torch.from_numpy(mk).to(DEV).to(dt),
                              torch.from_numpy(mv).to(DEV).to(dt))
    T = spec.tokens_per_agent
    pool = tk.PagedPool(spec.num_agents * T, spec.num_layers, spec.num_heads, spec.head_dim,
                        dtype=dt, device=DEV)
    maps = [pool.allocate(T, a) for a in range(spec.num_agents)]
    jobs = [j for a in range(spec.num_agents) for j in rounds.agent_jobs(spec, a, maps[a].slots)]
    col = tk.KVCollector(arena, pool)
    col.collect(col.plan(jobs))
    # V rows are bit copies of the master; K rows equal the oracle's rotation
    # of the (f32-upcast) master by the job's delta (rope_apply,
    # toymodel.py:60-83), sampled jobs x layers
    for n, j in enumerate(jobs[:: 37]):
        r0 = j.segment * spec.seg_len
        got_v = pool.v[:, torch.from_numpy(j.dst_rows).to(DEV)]
        assert torch.equal(got_v, arena.v[:, r0:r0 + spec.seg_len])
        for layer in (n % spec.num_layers, spec.num_layers - 1):
            got_k = pool.k[layer, torch.from_numpy(j.dst_rows).to(DEV)].float().cpu().numpy()
            master = arena.k[layer, r0:r0 + spec.seg_len].float().cpu().numpy()
            want = ref.rope_apply(master, np.broadcast_to(j.delta, (spec.seg_len,)))
            assert bf16_close(got_k, want) <= 1e-2
    # encode -> decode round trip of agent caches taken from the pool
    dense = []
    for m in maps[:3]:
        sl = torch.from_numpy(m.slots).to(DEV)
        dense.append(tk.LayeredKv(pool.k[:, sl].contiguous(), pool.v[:, sl].contiguous(),
                                  np.arange(T)))
    rng = np.random.default_rng(3)
    mirrors, hints = [], []
    for d in dense[1:]:
        mir = dense[0].copy()
        blocks = sorted(rng.choice(-(-T // 32), 15, replace=False).tolist())
        for b in blocks:
            mir.k[:, b * 32:(b + 1) * 32] = d.k[:, b * 32:(b + 1) * 32]
            mir.v[:, b * 32:(b + 1) * 32] = d.v[:, b * 32:(b + 1) * 32]
        mirrors.append(mir)
        hints.append(np.concatenate([np.arange(b * 32, min(T, b * 32 + 32)) for b in blocks]))
    diffs = tk.encode_batch(dense[0], mirrors, hints, tk.CacheBlockConfig(32))
    m32k, m32v = dense[0].k.float().cpu().numpy(), dense[0].v.float().cpu().numpy()
    for mir, h, diff in zip(mirrors, hints, diffs):
        # index lists bit-exact against the oracle on the upcast caches
        want = ref.encode_diff(m32k, m32v, mir.k.float().cpu().numpy(),
                               mir.v.float().cpu().numpy(), h, 32)
        assert [ld.indices.tolist() for ld in diff.layers] == [w.indices.tolist() for w in want]
        back = tk.diff_decode_dense(dense[0], diff)
        assert torch.equal(back.k, mir.k) and torch.equal(back.v, mir.v)


def test_slot_arena_planning_equals_row_planning():
    spec = rounds.CONFIGS["c2"].scaled(num_layers=2, num_agents=5, num_segments=4, hist_len=20)
    mk, mv = rounds.master_planes_host(spec)
    dt = spec.torch_dtype
    arena = rounds.make_arena(spec, torch.from_numpy(mk).to(DEV).to(dt),
                              torch.from_numpy(mv).to(DEV).to(dt))
    T = spec.tokens_per_agent
    pools = []
    for mode in ("rows", "offsets"):
        pool = tk.PagedPool(spec.num_agents * T + 100, spec.num_layers, spec.num_heads,
                            spec.head_dim, dtype=dt, device=DEV)
        pool.allocate(37)            # non-trivial slot maps
        maps = [pool.allocate(T, a) for a in range(spec.num_agents)]
        col = tk.KVCollector(arena, pool)
        if mode == "rows":
            plan = col.plan([j for a in range(spec.num_agents)
                             for j in rounds.agent_jobs(spec, a, maps[a].slots)])
        else:
            sa = tk.SlotArena(maps, DEV)
            plan = col.plan_offsets(*rounds.round_offsets(spec, range(spec.num_agents), sa.base),
                                    sa)
        col.collect(plan)
        pools.append((pool.k.clone(), pool.v.clone()))
    assert torch.equal(pools[0][0], pools[1][0]) and torch.equal(pools[0][1], pools[1][1])


def test_round_graph_replay_equals_eager_collect():
    """A captured round (CUDA graph: K0 + K1) replays to the same pool bytes
    as the eager launches, and reads the arena at replay time."""
    spec = rounds.CONFIGS["c2"].scaled(num_layers=3, num_agents=5, num_segments=4, hist_len=33)
    mk, mv = rounds.master_planes_host(spec)
    dt = spec.torch_dtype
    dev = torch.device("cuda", 0)
    arena = rounds.make_arena(spec, torch.from_numpy(mk).to(dev).to(dt),
                              torch.from_numpy(mv).to(dev).to(dt))
    T = spec.tokens_per_agent
    pools = []
    for _ in range(2):
        pool = tk.PagedPool(spec.num_agents * T, spec.num_layers, spec.num_heads, spec.head_dim,
                            dtype=dt, device=dev)
        maps = [pool.allocate(T, a) for a in range(spec.num_agents)]
        jobs = [j for a, m in enumerate(maps) for j in rounds.agent_jobs(spec, a, m.slots)]
        pools.append((pool, tk.KVCollector(arena, pool), jobs))
    (pa, ca, ja), (pb, cb, jb) = pools
    graph = cb.capture(cb.plan(jb))
    for step in range(3):
        arena.k.mul_(-1) if step else None          # new master contents every round
        ca.collect(ca.plan(ja))
        assert graph.replay() == (1 if graph.plan.fuse_table else 2)
        torch.cuda.synchronize()
        assert torch.equal(pa.k, pb.k) and torch.equal(pa.v, pb.v), step


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_replayed_plan_auto_graph_and_fused_table(dtype):
    """KVCollector.collect of the same plan again is captured as a CUDA graph
    (tdkv_collect_round) and replayed; every replay reads the arena as it is
    then.  The graphed run computes the cos/sin rows inside K1 (fused K0,
    one kernel per round), the reference run launches K0 + K1 plainly every
    round: the pools are bit-identical (same arithmetic), and the replays
    are counted as tdkv launches."""
    base = rounds.CONFIGS["c1"] if dtype == "f32" else rounds.CONFIGS["c2"]
    spec = base.scaled(num_layers=3, num_agents=6, num_segments=4, hist_len=21)
    mk, mv = rounds.master_planes_host(spec)
    dt = spec.torch_dtype
    arena = rounds.make_arena(spec, torch.from_numpy(mk).to(DEV).to(dt),
                              torch.from_numpy(mv).to(DEV).to(dt))
    T = spec.tokens_per_agent
    runs = []
    for auto in (True, False):
        pool = tk.PagedPool(spec.num_agents * T, spec.num_layers, spec.num_heads, spec.head_dim,
                            dtype=dt, device=DEV)
        maps = [pool.allocate(T, a) for a in range(spec.num_agents)]
        col = tk.KVCollector(arena, pool)
        col.auto_graph = auto
        plan = col.plan([j for a, m in enumerate(maps) for j in rounds.agent_jobs(spec, a, m.slots)])
        plan.fuse_table = auto           # before the first launch (the call is cached)
        runs.append((pool, col, plan, maps))
    for step in range(5):
        arena.k.mul_(-1) if step % 2 else arena.v.add_(1)     # new master contents every round
        outs = []
        for pool, col, plan, _ in runs:
            before = tk.launch_count()
            kernels = 1 if plan.fuse_table else 2
            assert col.collect(plan) == kernels
            assert tk.launch_count() - before == kernels
            torch.cuda.synchronize()
            outs.append((pool.k.clone(), pool.v.clone()))
        assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1]), step
    assert runs[0][1]._graph is not None and runs[1][1]._graph is None
    # and the graph-replayed pool still equals the oracle (f32: 1e-5)
    if dtype == "f32":
        pool, col, plan, maps = runs[0]
        gk = pool.k.cpu().numpy()
        ak = arena.k.cpu().numpy()
        for a, m in enumerate(maps):
            for j in rounds.agent_jobs(spec, a, m.slots):
                r0 = j.segment * spec.seg_len
                want = ref.rope_apply(ak[1, r0:r0 + spec.seg_len], j.delta)
                assert np.abs(gk[1, j.dst_rows] - want).max() <= F32_TOL


@pytest.mark.parametrize("dtype,heads,head_dim,agents", [
    ("bf16", 4, 128, 40),      # 40 jobs per tile: three job groups in the fused instantiation
    ("f32", 8, 64, 21),        # C1 rows, two groups
    ("f32", 1, 6, 9),          # 24-byte rows: 8-byte units, the generic kernel's fused path
    ("bf16", 3, 10, 17),       # 60-byte rows: 4-byte units, no TMA staging
])
def test_fused_table_equals_k0_table(dtype, heads, head_dim, agents):
    """A round collected with the cos/sin rows computed inside K1 (fused K0)
    equals the same round with K0's table, bit for bit, whatever the unit
    width, the job-group count per tile and the staging path; and matches the
    oracle (f32 within 1e-5)."""
    base = rounds.CONFIGS["c1"] if dtype == "f32" else rounds.CONFIGS["c2"]
    spec = base.scaled(num_layers=2, num_heads=heads, head_dim=head_dim, num_agents=agents,
                       num_segments=3, seg_len=40, hist_len=13)
    mk, mv = rounds.master_planes_host(spec)
    dt = spec.torch_dtype
    arena = rounds.make_arena(spec, torch.from_numpy(mk).to(DEV).to(dt),
                              torch.from_numpy(mv).to(DEV).to(dt))
    T = spec.tokens_per_agent
    outs = []
    for fused in (True, False):
        pool = tk.PagedPool(agents * T + 40, spec.num_layers, heads, head_dim, dtype=dt,
                            device=DEV)
        maps = [pool.allocate(T, a) for a in range(agents)]
        col = tk.KVCollector(arena, pool)
        col.auto_graph = False
        plan = col.plan([j for a, m in enumerate(maps) for j in rounds.agent_jobs(spec, a, m.slots)])
        plan.fuse_table = fused
        col.collect(plan)
        torch.cuda.synchronize()
        outs.append((pool.k.float().cpu().numpy(), pool.v.float().cpu().numpy(), maps))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    if dtype == "f32":
        gk, gv, maps = outs[0]
        for a, m in enumerate(maps):
            for j in rounds.agent_jobs(spec, a, m.slots):
                r0 = j.segment * spec.seg_len
                for layer in range(spec.num_layers):
                    want = ref.rope_apply(mk[layer, r0:r0 + spec.seg_len], j.delta)
                    assert np.abs(gk[layer, j.dst_rows] - want).max() <= F32_TOL
                    assert np.array_equal(gv[layer, j.dst_rows], mv[layer, r0:r0 + spec.seg_len])


@pytest.mark.parametrize("dtype,heads,head_dim,fused", [
    ("f32", 8, 64, True), ("f32", 8, 64, False),      # C1 rows: 2 KiB, 16 units per head
    ("bf16", 4, 128, True), ("bf16", 4, 128, False),  # C2 rows: 1 KiB
    ("bf16", 8, 128, False),                          # C3 rows: 2 KiB
    ("bf16", 16, 32, True),                           # 4 units per head
    ("f32", 2, 256, False),                           # 64 units per head
])
def test_collector_neox_pairs_match_oracle(dtype, heads, head_dim, fused):
    """KVCollector(rope_style="neox") rotates element j of a head with
    element j + D/2 (one thread owns both units of a pair) -- an extension
    beyond the reference's interleaved pairs -- and equals
    oracle.rope_apply_neox: f32 bit for bit, bf16 within the bf16
    tolerance; V is copied."""
    base = rounds.CONFIGS["c1"] if dtype == "f32" else rounds.CONFIGS["c2"]
    spec = base.scaled(num_layers=2, num_heads=heads, head_dim=head_dim, num_agents=19,
                       num_segments=3, seg_len=40, hist_len=13)
    mk, mv = rounds.master_planes_host(spec)
    dt = spec.torch_dtype
    arena = rounds.make_arena(spec, torch.from_numpy(mk).to(DEV).to(dt),
                              torch.from_numpy(mv).to(DEV).to(dt))
    if dtype == "bf16":           # the oracle sees the bf16 values the kernel reads
        mk = arena.k.float().cpu().numpy()
        mv = arena.v.float().cpu().numpy()
    T = spec.tokens_per_agent
    pool = tk.PagedPool(19 * T + 40, 2, heads, head_dim, dtype=dt, device=DEV)
    maps = [pool.allocate(T, a) for a in range(19)]
    col = tk.KVCollector(arena, pool, rope_style="neox")
    col.auto_graph = False
    plan = col.plan([j for a, m in enumerate(maps) for j in rounds.agent_jobs(spec, a, m.slots)])
    plan.fuse_table = fused
    col.collect(plan)
    torch.cuda.synchronize()
    gk, gv = pool.k.float().cpu().numpy(), pool.v.float().cpu().numpy()
    for a, m in enumerate(maps):
        for j in rounds.agent_jobs(spec, a, m.slots):
            r0 = j.segment * spec.seg_len
            for layer in range(2):
                want = ref.rope_apply_neox(mk[layer, r0:r0 + spec.seg_len], j.delta)
                got = gk[layer, j.dst_rows]
                if dtype == "f32":
                    assert np.array_equal(got, want)
                else:
                    assert np.abs(got - want).max() <= 1e-2 * max(1.0, np.abs(want).max())
                assert np.array_equal(gv[layer, j.dst_rows], mv[layer, r0:r0 + spec.seg_len])
    # the interleaved form differs (the pairing is not a no-op)
    col2 = tk.KVCollector(arena, pool)
    col2.collect(col2.plan([j for a, m in enumerate(maps)
                            for j in rounds.agent_jobs(spec, a, m.slots)]))
    torch.cuda.synchronize()
    assert not np.array_equal(pool.k.float().cpu().numpy(), gk)


def test_collector_neox_rejects_unsupported_layouts():
    """Half a head must be whole 16-byte units (f32 head_dim 4: 8 bytes); the
    chunked launch paths refuse rotate-half plans rather than rotate them
    interleaved."""
    spec = rounds.CONFIGS["c1"].scaled(num_layers=1, num_heads=2, head_dim=4, num_agents=2,
                                       num_segments=1, seg_len=8, hist_len=3)
    mk, mv = rounds.master_planes_host(spec)
    arena = rounds.make_arena(spec, torch.from_numpy(mk).to(DEV), torch.from_numpy(mv).to(DEV))
    T = spec.tokens_per_agent
    pool = tk.PagedPool(2 * T, 1, 2, 4, device=DEV)
    maps = [pool.allocate(T, a) for a in range(2)]
    col = tk.KVCollector(arena, pool, rope_style="neox")
    plan = col.plan([j for a, m in enumerate(maps) for j in rounds.agent_jobs(spec, a, m.slots)])
    with pytest.raises(tk.TdkvError, match="NeoX"):
        col.collect(plan)
    with pytest.raises(ValueError, match="neox"):
        plan.launch_collect(arena, pool.k, pool.v, pool.layer_stride)
    with pytest.raises(ValueError, match="rope_style"):
        tk.KVCollector(arena, pool, rope_style="gptj")


@pytest.mark.parametrize("heads,dim", [(1, 64), (3, 64), (8, 128), (2, 256), (5, 32)])
@pytest.mark.parametrize("style", ["interleaved", "neox"])
@pytest.mark.parametrize("fuse", ["0", "1"])
def test_paired_loop_geometries_bf16_against_oracle(heads, dim, style, fuse, monkeypatch):
    """bfloat16 rounds run K1's paired loop (two 16-byte units per thread,
    K0 rows staged per job group): odd head counts, head_dim 32-256, a job
    whose delta varies per row (per-row table rows, not staged), jobs of
    several segments and more jobs per tile than one group holds -- every
    rotated key within 1e-2 of the oracle on the bf16-rounded masters, V
    bit for bit."""
    from paper_2604_03143_b200 import collector as col_mod
    # "0": K0's table (the paired loop with staged rows); "1": the fused table
    monkeypatch.setattr(col_mod, "_FUSE_TABLE", fuse)
    rng = np.random.default_rng(heads * 1000 + dim)
    L, n_seg, seg = 2, 3, 37
    mk = rng.standard_normal((L, n_seg * seg, heads, dim)).astype(np.float32)
    mv = rng.standard_normal((L, n_seg * seg, heads, dim)).astype(np.float32)
    mk_b = torch.from_numpy(mk).to(DEV).bfloat16()
    mv_b = torch.from_numpy(mv).to(DEV).bfloat16()
    pos = [np.arange(s * 50, s * 50 + seg) for s in range(n_seg)]
    arena = tk.MasterArena(mk_b, mv_b, np.arange(n_seg) * seg, np.full(n_seg, seg), pos)
    jobs = []
    for j in range(40):                          # > 16 jobs per master tile
        s = j % n_seg
        if j == 7 and fuse == "0":               # per-row deltas (table rows not staged)
            delta = rng.integers(-300, 300, seg)
        else:
            delta = np.full(seg, int(rng.integers(-500, 2000)))
        jobs.append(tk.CollectJob(s, np.arange(j * seg, (j + 1) * seg), delta))
    rows = 40 * seg
    pool = tk.PagedPool(rows + 8, L, heads, dim, dtype=torch.bfloat16, device=DEV)
    col = tk.KVCollector(arena, pool, 10000.0, rope_style=style)
    plan = col.plan(jobs)
    assert plan.fuse_table == (fuse == "1")
    col.collect(plan)
    got_k = pool.k.float().cpu().numpy()
    got_v = pool.v.float().cpu().numpy()
    mk32 = mk_b.float().cpu().numpy()
    mv32 = mv_b.float().cpu().numpy()
    rope = ref.rope_apply if style == "interleaved" else ref.rope_apply_neox
    for j, job in enumerate(jobs):
        r0 = job.segment * seg
        dst = job.dst_rows
        for layer in range(L):
            want = rope(mk32[layer, r0:r0 + seg], job.delta)
            assert np.abs(got_k[layer, dst] - want).max() <= 1e-2 * max(1.0, np.abs(want).max())
            assert np.array_equal(got_v[layer, dst], mv32[layer, r0:r0 + seg])
