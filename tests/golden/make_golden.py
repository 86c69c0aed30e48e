"""Generate golden vectors from the reference package itself.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports ``roundkv`` 0.1.0 read-only from ``/root/reference/pkg/src`` and
records the reference's own outputs for the hot-path functions into small
fixtures next to this script.  The fixtures are committed; nothing that runs
on the GPU box reads ``/root/reference``.

Inputs are regenerated from seeds wherever possible (numpy's PCG64 streams
are platform-stable), so most fixtures hold only seeds plus the reference's
integer outputs and SHA-256 digests of its float outputs.  Small realistic
caches produced by the reference's toy model (which the oracle does not
restate) are stored verbatim in ``family.npz``.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from types import SimpleNamespace

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from roundkv.collective import collective_recover, form_groups  # noqa: E402
from roundkv.core import CacheBlockConfig, LayeredKv, ModelConfig, PositionSpan, token_digest  # noqa: E402
from roundkv.diffstore import (  # noqa: E402
    DiffStore, HintSoundnessError, MasterEntry, MirrorHandle, encode_diff,
    serialize_diff,
)
from roundkv.ledger import CostLedger  # noqa: E402
from roundkv.paged_pool import PagedPool  # noqa: E402
from roundkv.collective import select_master  # noqa: E402
from roundkv.pic import (PicConfig, _skeleton, align_cached, key_diff,  # noqa: E402
                         prepare_request, probe_and_select, recover_prepared)
from roundkv.toymodel import _selective_forward  # noqa: E402
from roundkv.restore import dense_restore, fused_restore  # noqa: E402
from roundkv.segment_index import SegmentCacheEntry, SegmentIndex  # noqa: E402
from roundkv.toymodel import build_weights, full_prefill, rope_apply  # noqa: E402
from roundkv.workload import WorkloadSpec, decode_context, generate_round  # noqa: E402
from roundkv.core import token_digest  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def random_kv(rng, t, layers, heads, dim, start=0):
    shape = (layers, t, heads, dim)
    return LayeredKv(rng.standard_normal(shape).astype(np.float32),
                     rng.standard_normal(shape).astype(np.float32),
                     np.arange(start, start + t, dtype=np.int64))


# ---------------------------------------------------------------------------


def gen_rope():
    """rope_apply on seeded K with deltas spanning +-8192 (toymodel.py:60-83)."""
    cases = []
    for seed, (t, h, d) in enumerate([(40, 2, 8), (33, 3, 16), (64, 2, 64), (17, 4, 128)]):
        rng = np.random.default_rng(1000 + seed)
        k = rng.standard_normal((t, h, d)).astype(np.float32)
        pos = rng.integers(-8192, 8192, t).astype(np.int64)
        cases.append({"seed": 1000 + seed, "shape": [t, h, d],
                      "sha": sha(rope_apply(k, pos, 10000.0))})
    return cases


def gen_collector():
    """A reference round through prepare_request + _skeleton + align_cached:
    the K rows the Collector produces and the V rows it copies."""
    model = ModelConfig(num_layers=2, num_heads=2, head_dim=16, vocab_size=512,
                        weight_seed=5)
    weights = build_weights(model)
    spec = WorkloadSpec(num_agents=4, num_rounds=1, history_len=(9, 9, 9, 9),
                        shared_block_len=11, token_seed=3, permutation_seed=8)
    rnd = generate_round(spec, model, 0)
    index = SegmentIndex(budget_bytes=1 << 30)
    masters = []
    for agent, seg in enumerate(rnd.shared_outputs):
        ctx = decode_context(spec, model, 0, agent)
        stream = list(ctx) + [model.separator_token] + list(seg.tokens)
        kv = full_prefill(weights, stream)
        lo = len(ctx) + 1
        rows = LayeredKv(kv.k[:, lo:].copy(), kv.v[:, lo:].copy(), kv.positions[lo:].copy())
        index.insert(SegmentCacheEntry(seg.digest, rows.positions, SimpleNamespace(kv=rows),
                                       token_digest(ctx), rows.dense_nbytes))
        masters.append(rows)
    preps = [prepare_request(rnd.prompts[a], model, index, request_id=a) for a in range(4)]
    contexts = [_skeleton(weights, p) for p in preps]
    ledger = CostLedger(model.num_layers)
    align_cached(preps, contexts, model.rope_base, ledger)
    arrays = {}
    meta = {"rope_calls_by_layer": ledger.rope_calls_by_layer, "agents": []}
    for i, m in enumerate(masters):
        arrays[f"master{i}_k"] = m.k
        arrays[f"master{i}_v"] = m.v
        arrays[f"master{i}_pos"] = m.positions
    for a, (p, (ck, cv)) in enumerate(zip(preps, contexts)):
        hits = []
        for h in p.hits:
            src = masters.index(h.kv)
            hits.append({"master": src, "target": h.target_idx.tolist(),
                         "delta": h.delta.tolist()})
        shared = p.shared_idx
        arrays[f"agent{a}_k_shared"] = ck[:, shared]
        arrays[f"agent{a}_v_shared"] = cv[:, shared]
        meta["agents"].append({"T": int(p.num_tokens), "hits": hits,
                               "shared_idx": shared.tolist()})
    # the check-layer selection on the same round (pic.probe_and_select):
    # fresh probe keys, cached (aligned) keys, and the reference's outputs
    pic = PicConfig(recompute_fraction=0.15, check_layer=1)
    fresh_rows, cached_rows, counts = [], [], []
    for p, (ck, cv) in zip(preps, contexts):
        shared = p.shared_idx
        fix = np.union1d(shared, p.structural_idx)
        k, _ = _selective_forward(weights, p.tokens, p.positions, fix, ck, cv,
                                  max_layer=pic.check_layer + 1)
        fresh_rows.append(k[pic.check_layer][np.searchsorted(fix, shared)])
        cached_rows.append(ck[pic.check_layer][shared])
        counts.append(int(shared.size))
    sel = probe_and_select(weights, preps, contexts, pic, CostLedger(model.num_layers))
    arrays["sel_fresh"] = np.concatenate(fresh_rows)
    arrays["sel_cached"] = np.concatenate(cached_rows)
    arrays["sel_mags"] = key_diff(arrays["sel_fresh"], arrays["sel_cached"])
    meta["selection"] = {
        "fraction": pic.recompute_fraction, "counts": counts,
        "important": [imp.tolist() for imp, _ in sel],
        "important_rel": [np.searchsorted(p.shared_idx, imp).tolist()
                          for p, (imp, _) in zip(preps, sel)],
        "deviation": [dev for _, dev in sel],
        "master": int(select_master({i: d for i, (_, d) in enumerate(sel)})),
    }
    np.savez_compressed(os.path.join(HERE, "collector.npz"), **arrays)
    return meta


def gen_family():
    """collective_recover -> encode_family -> fused/dense restore on a small
    toy-model round: the realistic diff inputs and the reference's outputs."""
    model = ModelConfig(num_layers=3, num_heads=2, head_dim=8, vocab_size=512, weight_seed=21)
    weights = build_weights(model)
    spec = WorkloadSpec(num_agents=3, num_rounds=1, history_len=12, shared_block_len=6,
                        token_seed=31, permutation_seed=None)
    rnd = generate_round(spec, model, 0)
    index = SegmentIndex(budget_bytes=1 << 30)
    for agent, seg in enumerate(rnd.shared_outputs):
        ctx = decode_context(spec, model, 0, agent)
        stream = list(ctx) + [model.separator_token] + list(seg.tokens)
        kv = full_prefill(weights, stream)
        lo = len(ctx) + 1
        rows = LayeredKv(kv.k[:, lo:].copy(), kv.v[:, lo:].copy(), kv.positions[lo:].copy())
        index.insert(SegmentCacheEntry(seg.digest, rows.positions, SimpleNamespace(kv=rows),
                                       token_digest(ctx), rows.dense_nbytes))
    preps = [prepare_request(rnd.prompts[a], model, index, request_id=a) for a in range(3)]
    groups, _ = form_groups(preps)
    blocks = CacheBlockConfig(block_size=8)
    results, plan = collective_recover(weights, groups[0], PicConfig(0.15, 1))
    store = DiffStore(blocks)
    enc = store.encode_family(plan, results)
    arrays = {}
    meta = {"master_id": int(plan.master_id), "block_size": 8, "rope_base": model.rope_base,
            "stats": {"dense": enc.stats.dense_nbytes,
                      "payload": enc.stats.diff_payload_nbytes,
                      "serialized": enc.stats.diff_serialized_nbytes,
                      "changed": enc.stats.changed_blocks,
                      "ratios": enc.stats.ratios,
                      "family_cost": enc.stats.family_cost},
            "mirrors": []}
    arrays["master_k"] = results[plan.master_id].kv.k
    arrays["master_v"] = results[plan.master_id].kv.v
    arrays["positions"] = results[plan.master_id].kv.positions
    for rid, handle in sorted(enc.mirrors.items()):
        arrays[f"mirror{rid}_k"] = results[rid].kv.k
        arrays[f"mirror{rid}_v"] = results[rid].kv.v
        arrays[f"hints{rid}"] = plan.mirror_diff_hints[rid]
        wire = serialize_diff(handle.diff)
        T = handle.master.kv.num_tokens
        pool = PagedPool(4 * T + 32, 3, 2, 8, block_size=8)
        fmap = pool.allocate(T, 1)
        dmap = pool.allocate(T, 2)
        span = PositionSpan.shifted(handle.positions, 16)
        led = CostLedger(3)
        fused_restore(handle, span, pool, fmap, model.rope_base, ledger=led)
        dense_restore(handle, span, pool, dmap, model.rope_base)
        fk = np.stack([pool.read_rows(fmap, l)[0] for l in range(3)])
        fv = np.stack([pool.read_rows(fmap, l)[1] for l in range(3)])
        meta["mirrors"].append({
            "rid": int(rid),
            "indices": [ld.indices.tolist() for ld in handle.diff.layers],
            "wire_sha": hashlib.sha256(wire).hexdigest(),
            "wire_len": len(wire),
            "fused_slots": fmap.slots.tolist(),
            "fused_sha": sha(fk, fv),
            "bytes_moved": led.bytes_moved,
            "temp_peak": led.temp_buffer_peak_bytes,
        })
    np.savez_compressed(os.path.join(HERE, "family.npz"), **arrays)
    return meta


def _perturb(rng, master, blocks, block_ids):
    mirror = master.copy()
    hints = []
    for b in block_ids:
        lo, hi = blocks.block_bounds(b, master.num_tokens)
        mirror.k[:, lo:hi] = rng.standard_normal(mirror.k[:, lo:hi].shape).astype(np.float32)
        mirror.v[:, lo:hi] = rng.standard_normal(mirror.v[:, lo:hi].shape).astype(np.float32)
        hints.extend(range(lo, hi))
    return mirror, np.asarray(sorted(hints), dtype=np.int64)


def gen_codec_trials():
    """C04-style randomized encode trials (acceptance test_c04) regenerated
    from a seed; records indices, wire length and digest per trial."""
    out = []
    rng = np.random.default_rng(0xD1FF)
    for trial in range(1000):          # the acceptance C04 count
        bs = int(rng.choice([8, 16, 32]))
        blocks = CacheBlockConfig(block_size=bs)
        t = int(rng.integers(1, 180))
        layers = int(rng.integers(1, 4))
        heads = int(rng.integers(1, 3))
        dim = 2 * int(rng.integers(1, 5))
        start = int(rng.integers(0, 40))
        master = random_kv(rng, t, layers, heads, dim, start=start)
        mirror = master.copy()
        nb = blocks.num_blocks(t)
        count = int(rng.integers(0, nb + 1))
        chosen = rng.choice(nb, size=count, replace=False)
        hints = []
        for b in sorted(int(b) for b in chosen):
            lo, hi = blocks.block_bounds(b, t)
            hints.extend(range(lo, hi))
            mode = int(rng.integers(0, 4))
            row = int(rng.integers(lo, hi))
            if mode == 0:
                mirror.k[:, lo:hi] += 1.0
            elif mode == 1:
                mirror.v[:, lo:hi] -= 1.0
            elif mode == 2:
                mirror.k[:, row] = rng.standard_normal(mirror.k[:, row].shape).astype(np.float32)
        diff = encode_diff(master, mirror, np.asarray(hints, dtype=np.int64), blocks)
        wire = serialize_diff(diff)
        out.append({"indices": [ld.indices.tolist() for ld in diff.layers],
                    "wire_len": len(wire), "wire_sha": hashlib.sha256(wire).hexdigest()})
    return out


# (plane, index, value or None = +2.5, edit the master instead of the mirror)
VIOLATION_CASES = {
    "nan_k": [("k", (0, 100, 0, 0), float("nan"), False)],
    "nan_v_and_k": [("v", (0, 100, 0, 0), float("nan"), False), ("k", (0, 101, 1, 3), None, False)],
    "nan_both_v": [("v", (2, 99, 1, 1), float("nan"), False), ("v", (2, 99, 1, 1), float("nan"), True)],
    "neg_inf_k": [("k", (3, 127, 0, 7), float("-inf"), False)],
    "signed_zero": [("k", (1, 110, 1, 2), 0.0, True), ("k", (1, 110, 1, 2), -0.0, False)],
}


def gen_known_answers():
    """The worked examples of test_diffstore.py / acceptance C07."""
    blocks = CacheBlockConfig(block_size=32)
    res = {}
    rng = np.random.default_rng(11)
    master = random_kv(rng, 640, 4, 2, 8)
    mirror, hints = _perturb(rng, master, blocks, [3, 17])
    diff = encode_diff(master, mirror, hints, blocks)
    wire = serialize_diff(diff)
    res["worked"] = {"seed": 11, "payload": diff.payload_nbytes, "dense": master.dense_nbytes,
                     "wire_len": len(wire), "wire_sha": hashlib.sha256(wire).hexdigest(),
                     "changed": diff.changed_blocks_per_layer}
    rng = np.random.default_rng(24)
    master = random_kv(rng, 128, 4, 2, 8)
    mirror, hints = _perturb(rng, master, blocks, [1])
    mirror.v[0, 100, 0, 0] += 0.5
    try:
        encode_diff(master, mirror, hints, blocks)
        raise AssertionError("expected a soundness error")
    except HintSoundnessError as exc:
        res["violation"] = {"seed": 24, "message": str(exc)}
    # the violation magnitude with NaN / inf outside the hints: numpy's max
    # propagates NaN within a plane, Python's max(k, v) keeps K's NaN and drops
    # V's (diffstore.py:157-160)
    res["violation_special"] = []
    for case, edits in VIOLATION_CASES.items():
        rng = np.random.default_rng(24)
        master = random_kv(rng, 128, 4, 2, 8)
        mirror, hints = _perturb(rng, master, blocks, [1])
        for plane, idx, value, on_master in edits:
            tgt = master if on_master else mirror
            getattr(tgt, plane)[idx] = value if value is not None else \
                getattr(tgt, plane)[idx] + 2.5
        try:
            encode_diff(master, mirror, hints, blocks)
            message = None
        except HintSoundnessError as exc:
            message = str(exc)
        res["violation_special"].append({"case": case, "message": message})
    rng = np.random.default_rng(21)
    master = random_kv(rng, 70, 4, 2, 8)
    mirror, hints = _perturb(rng, master, blocks, [2])
    wire = serialize_diff(encode_diff(master, mirror, hints, blocks))
    res["partial"] = {"seed": 21, "wire_sha": hashlib.sha256(wire).hexdigest(),
                      "wire_len": len(wire)}
    return res


def gen_restores():
    """C05-style fused restores (acceptance test_c05): pool digests."""
    out = []
    rng = np.random.default_rng(0xF05E)
    blocks = CacheBlockConfig(block_size=16)
    for trial in range(200):           # the acceptance C05 count
        t = int(rng.integers(8, 90))
        start = int(rng.integers(0, 60))
        delta = int(rng.integers(-start, 80))
        master_kv = random_kv(rng, t, 3, 2, 8, start=start)
        nb = blocks.num_blocks(t)
        count = int(rng.integers(0, min(nb, 3) + 1))
        chosen = sorted(int(b) for b in rng.choice(nb, count, replace=False))
        mirror_kv, hints = _perturb(rng, master_kv, blocks, chosen)
        diff = encode_diff(master_kv, mirror_kv, hints, blocks)
        master = MasterEntry(0, master_kv)
        master.pin_count = 1
        handle = MirrorHandle(0, trial, master, diff)
        span = PositionSpan.shifted(master_kv.positions, delta)
        pool = PagedPool(128, 3, 2, 8, block_size=16)
        smap = pool.allocate(t, request_id=trial)
        led = CostLedger(3)
        fused_restore(handle, span, pool, smap, 10000.0, ledger=led)
        k = np.stack([pool.read_rows(smap, l)[0] for l in range(3)])
        v = np.stack([pool.read_rows(smap, l)[1] for l in range(3)])
        out.append({"t": t, "delta": delta, "slots": smap.slots.tolist(),
                    "sha": sha(k, v), "bytes_moved": led.bytes_moved})
    return out


def gen_allocator():
    """A seeded allocate/free stream through PagedPool (paged_pool.py:106-148)."""
    pool = PagedPool(256, 1, 1, 2, block_size=32, debug=False)
    rng = np.random.default_rng(7)
    live, ops = [], []
    for step in range(300):
        if live and (rng.random() < 0.45 or pool.free_count < 20):
            i = int(rng.integers(len(live)))
            m = live.pop(i)
            pool.free(m)
            ops.append({"op": "free", "serial": m.serial})
        else:
            n = int(rng.integers(1, 40))
            if n > pool.free_count:
                ops.append({"op": "skip", "n": n})
                continue
            m = pool.allocate(n, request_id=step)
            live.append(m)
            ops.append({"op": "alloc", "n": n, "serial": m.serial, "slots": m.slots.tolist()})
    return ops


def gen_segment_index():
    """A seeded insert / lookup / pin / remove / evict stream through
    segment_index.SegmentIndex (segment_index.py:86-183); entries are
    labelled by creation order, state recorded after every step."""
    from roundkv.segment_index import PinnedEntryError, SegmentCacheEntry, SegmentIndex

    class Ref:
        def __init__(self):
            self.pinned = False

    rng = np.random.default_rng(23)
    made, label = [], {}
    evicted = []
    idx = SegmentIndex(2000, is_pinned=lambda r: r.pinned,
                       on_evict=lambda e: evicted.append(label[id(e)]))
    ops = []
    for _ in range(1500):
        r = int(rng.integers(0, 10))
        if r < 4:
            tok, nb = int(rng.integers(0, 30)), int(rng.integers(1, 300))
            e = SegmentCacheEntry(token_digest([tok]), np.arange(1), Ref(), b"c" * 16, nb)
            label[id(e)] = len(made)
            made.append(e)
            idx.insert(e)
            op = {"op": "insert", "tok": tok, "nbytes": nb}
        elif r < 7:
            tok = int(rng.integers(0, 30))
            hit = idx.lookup(token_digest([tok]))
            op = {"op": "lookup", "tok": tok, "hit": -1 if hit is None else label[id(hit)]}
        elif r == 7 and made:
            i = int(rng.integers(0, len(made)))
            made[i].kv_ref.pinned = not made[i].kv_ref.pinned
            op = {"op": "pin", "label": i}
        elif r == 8 and made:
            i = int(rng.integers(0, len(made)))
            try:
                idx.remove(made[i])
                op = {"op": "remove", "label": i, "raised": False}
            except PinnedEntryError:
                op = {"op": "remove", "label": i, "raised": True}
        else:
            b = int(rng.integers(0, 3000))
            op = {"op": "evict", "budget": b, "n": idx.evict_to_budget(b)}
        op.update(evicted=list(evicted), total=idx.total_bytes, len=len(idx),
                  lru=[label[id(e)] for e in idx.entries()])
        ops.append(op)
    return ops


def gen_toymodel():
    """Toy transformer outputs (the selective recompute's arithmetic,
    toymodel.py:36-192): weights digests, a full prefill and a selective
    forward over a perturbed context, recorded verbatim (small)."""
    out = {}
    arrays = {}
    for name, (L, H, D, V, seed) in {"small": (3, 2, 8, 512, 21),
                                     "c1": (2, 8, 64, 1024, 0)}.items():
        cfg = ModelConfig(num_layers=L, num_heads=H, head_dim=D, vocab_size=V, weight_seed=seed)
        w = build_weights(cfg)
        rng = np.random.default_rng(100 + L)
        toks = [int(t) for t in rng.integers(0, V - 1, 48)]
        pre = full_prefill(w, toks)
        ctx_k = pre.k + rng.standard_normal(pre.k.shape).astype(np.float32) * 0.01
        ctx_v = pre.v + rng.standard_normal(pre.v.shape).astype(np.float32) * 0.01
        fix = np.sort(rng.choice(48, 13, replace=False)).astype(np.int64)
        pos = np.arange(48, dtype=np.int64) + 5
        k, v = _selective_forward(w, np.asarray(toks), pos, fix, ctx_k, ctx_v)
        k1, v1 = _selective_forward(w, np.asarray(toks), pos, fix, ctx_k, ctx_v, max_layer=1)
        out[name] = {"config": [L, H, D, V, seed],
                     "weights_sha": sha(w.embed, w.wq, w.wk, w.wv, w.wm),
                     "prefill_sha": sha(pre.k, pre.v), "selective_sha": sha(k, v),
                     "probe_sha": sha(k1, v1)}
        arrays[f"{name}_tokens"] = np.asarray(toks)
        arrays[f"{name}_ctx_k"] = ctx_k
        arrays[f"{name}_ctx_v"] = ctx_v
        arrays[f"{name}_fix"] = fix
        arrays[f"{name}_prefill_k"] = pre.k
        arrays[f"{name}_prefill_v"] = pre.v
        arrays[f"{name}_sel_k"] = k
        arrays[f"{name}_sel_v"] = v
    np.savez_compressed(os.path.join(HERE, "toymodel.npz"), **arrays)
    return out


def gen_recovery():
    """collective_recover (and serial recover_prepared) on two decode-seeded
    rounds: everything a duck-typed PreparedRequest needs, and the
    reference's results (caches, important sets, deviations, master, hints)."""
    meta = {}
    arrays = {}
    for case, (agents, perm_seed, hist, blen) in {"same_order": (3, None, 12, 6),
                                                  "permuted": (4, 17, 9, 7)}.items():
        model = ModelConfig(num_layers=3, num_heads=2, head_dim=8, vocab_size=512,
                            weight_seed=21)
        weights = build_weights(model)
        spec = WorkloadSpec(num_agents=agents, num_rounds=1, history_len=hist,
                            shared_block_len=blen, token_seed=31, permutation_seed=perm_seed)
        rnd = generate_round(spec, model, 0)
        index = SegmentIndex(budget_bytes=1 << 30)
        seg_rows = []
        for agent, seg in enumerate(rnd.shared_outputs):
            ctx = decode_context(spec, model, 0, agent)
            stream = list(ctx) + [model.separator_token] + list(seg.tokens)
            kv = full_prefill(weights, stream)
            lo = len(ctx) + 1
            rows = LayeredKv(kv.k[:, lo:].copy(), kv.v[:, lo:].copy(), kv.positions[lo:].copy())
            index.insert(SegmentCacheEntry(seg.digest, rows.positions, SimpleNamespace(kv=rows),
                                           token_digest(ctx), rows.dense_nbytes))
            seg_rows.append(rows)
            arrays[f"{case}_seg{agent}_k"] = rows.k
            arrays[f"{case}_seg{agent}_v"] = rows.v
            arrays[f"{case}_seg{agent}_pos"] = rows.positions
        preps = [prepare_request(rnd.prompts[a], model, index, request_id=a)
                 for a in range(agents)]
        groups, _ = form_groups(preps)
        pic = PicConfig(0.15, 1)
        results, plan = collective_recover(weights, groups[0], pic, CostLedger(3))
        serial = recover_prepared(weights, preps[0], pic, CostLedger(3))
        m = {"agents": agents, "members": [], "master_id": int(plan.master_id),
             "fraction": 0.15, "check_layer": 1, "model": [3, 2, 8, 512, 21]}
        for p in preps:
            rid = p.request_id
            for name in ("tokens", "positions", "private_idx", "structural_idx", "label_entry",
                         "label_offset"):
                arrays[f"{case}_r{rid}_{name}"] = np.asarray(getattr(p, name))
            arrays[f"{case}_r{rid}_k"] = results[rid].kv.k
            arrays[f"{case}_r{rid}_v"] = results[rid].kv.v
            m["members"].append({
                "rid": rid,
                "hits": [{"seg": seg_rows.index(h.kv), "target": h.target_idx.tolist()}
                         for h in p.hits],
                "important": plan.important[rid].tolist(),
                "deviation": plan.deviation_scores[rid],
                "hints": (plan.mirror_diff_hints[rid].tolist()
                          if rid in plan.mirror_diff_hints else None),
                "num_recomputed": results[rid].num_recomputed,
            })
        arrays[f"{case}_serial0_k"] = serial.kv.k
        arrays[f"{case}_serial0_v"] = serial.kv.v
        meta[case] = m
    np.savez_compressed(os.path.join(HERE, "recovery.npz"), **arrays)
    return meta


T3_CASES = {
    # two groups (history lengths 12 / 9) and a singleton remainder (20)
    "roomy": dict(history=(12, 12, 12, 9, 9, 9, 20), capacity=4096),
    # the same rounds in a pool too small for the restore verification
    "tight": dict(history=(12, 12, 12, 9, 9, 9, 20), capacity=470),
}


def gen_t3():
    """The reference's own T3 rounds (trace._run_t3, trace.py:332-403, via
    run_trace): the report rows -- ledger counters, compression lists,
    fidelity, restores verified -- plus every input a replay through another
    implementation of the hot path needs (the prepared requests of each group
    and of the remainder, the seeded segment rows, the oracle caches).  The
    prepared requests are captured by wrapping the reference's own calls;
    nothing about the control flow is restated here."""
    import roundkv.trace as trace
    from roundkv.core import flatten_prompt
    from roundkv.pic import PicConfig as _Pic
    from roundkv.trace import SimulationSpec, run_trace
    meta, arrays = {}, {}
    for case, cfg in T3_CASES.items():
        model = ModelConfig(num_layers=3, num_heads=2, head_dim=8, vocab_size=512,
                            weight_seed=21)
        wl = WorkloadSpec(num_agents=len(cfg["history"]), num_rounds=2,
                          history_len=cfg["history"], shared_block_len=6, token_seed=31,
                          permutation_seed=17)
        spec = SimulationSpec(model=model, workload=wl, pic=_Pic(0.15, 1),
                              blocks=CacheBlockConfig(8), pool_capacity_tokens=cfg["capacity"])
        seen = {"seeds": [], "groups": [], "remainder": []}
        real_seeds, real_cr, real_rp = trace._round_seeds, trace.collective_recover, \
            trace.recover_prepared

        def seeds_hook(spec_, weights_, rnd_):
            out = real_seeds(spec_, weights_, rnd_)
            seen["seeds"].append((rnd_.round_id, out))
            return out

        def cr_hook(weights_, group, pic_, ledger_=None):
            res, plan = real_cr(weights_, group, pic_, ledger_)
            seen["groups"].append((list(group.members), plan))
            return res, plan

        def rp_hook(weights_, prep, pic_, ledger_=None):
            seen["remainder"].append(prep)
            return real_rp(weights_, prep, pic_, ledger_)

        trace._round_seeds, trace.collective_recover, trace.recover_prepared = \
            seeds_hook, cr_hook, rp_hook
        try:
            report = run_trace(spec, paths=("T3",))
        finally:
            trace._round_seeds, trace.collective_recover, trace.recover_prepared = \
                real_seeds, real_cr, real_rp
        # seeded segment rows, keyed by the digest the hits resolve to
        seed_key = {}
        for rnd_id, seeds in seen["seeds"]:
            for a, (seg, rows, _ctx) in enumerate(seeds):
                key = f"{case}_seed_r{rnd_id}_a{a}"
                seed_key[seg.digest] = key
                arrays[key + "_k"], arrays[key + "_v"] = rows.k, rows.v
                arrays[key + "_pos"] = rows.positions
                arrays[key + "_tokens"] = np.asarray(seg.tokens, np.int64)

        def prep_meta(prep, tag):
            for name in ("tokens", "positions", "private_idx", "structural_idx",
                         "label_entry", "label_offset"):
                arrays[f"{tag}_{name}"] = np.asarray(getattr(prep, name))
            # the prompt layout itself (for the native prepare_request parity)
            segs = prep.layout.segments
            arrays[f"{tag}_layout_kinds"] = np.array([s.kind.value for s in segs])
            arrays[f"{tag}_layout_lens"] = np.array([len(s) for s in segs], np.int64)
            arrays[f"{tag}_layout_tokens"] = np.concatenate(
                [np.asarray(s.tokens, np.int64) for s in segs])
            ent_key = {}
            for h in prep.hits:
                ent_key[int(h.entry.entry_id)] = seed_key[h.entry.digest]
            arrays[f"{tag}_label_seed"] = np.array(
                [ent_key.get(int(e), "") for e in prep.label_entry])
            return {"rid": int(prep.request_id), "tag": tag, "agent": int(prep.layout.agent_id),
                    "slots": None if prep.slot_map is None else prep.slot_map.slots.tolist(),
                    "hits": [{"seed": seed_key[h.entry.digest], "target": h.target_idx.tolist()}
                             for h in prep.hits]}

        rounds_meta = []
        gi = ri = 0
        for row in report["rows"]:
            rnd = generate_round(wl, model, row["round"])
            weights = build_weights(model)
            for a, p in enumerate(rnd.prompts):
                o = full_prefill(weights, flatten_prompt(p, model.separator_token))
                arrays[f"{case}_oracle_r{row['round']}_a{a}_k"] = o.k
                arrays[f"{case}_oracle_r{row['round']}_a{a}_v"] = o.v
            groups = []
            for _ in range(row["num_groups"]):
                members, plan = seen["groups"][gi]
                groups.append({
                    "members": [prep_meta(m, f"{case}_g{gi}_r{m.request_id}") for m in members],
                    "master_id": int(plan.master_id),
                    "hints": {str(k): v.tolist() for k, v in plan.mirror_diff_hints.items()}})
                gi += 1
            remainder = []
            for _ in range(row["num_remainder"]):
                prep = seen["remainder"][ri]
                remainder.append(prep_meta(prep, f"{case}_rem{ri}_r{prep.request_id}"))
                ri += 1
            rounds_meta.append({
                "round": row["round"],
                "prompts": [[int(p.agent_id), len(flatten_prompt(p, model.separator_token))]
                            for p in rnd.prompts],
                "seeds": [f"{case}_seed_r{row['round']}_a{a}"
                          for a in range(len(rnd.shared_outputs))],
                "groups": groups, "remainder": remainder, "row": row})
        meta[case] = {"model": [3, 2, 8, 512, 21], "block_size": 8,
                      "capacity": cfg["capacity"], "restore_shift": spec.restore_shift,
                      "fraction": 0.15, "check_layer": 1, "rounds": rounds_meta}
    np.savez_compressed(os.path.join(HERE, "t3.npz"), **arrays)
    return meta


def _prepare_world():
    """A segment index of named entries and prompts exercising every branch
    of prepare_request (pic.py:110-163): hits, a miss, a task segment, a
    digest with two entries (the most recent wins), a repeated segment, a
    private-only prompt.  Shared by gen_prepare and the parity tests (which
    rebuild the same world from the recorded names and tokens)."""
    from roundkv.core import PromptLayout, Segment, SegmentKind
    rng = np.random.default_rng(404)
    toks = {n: tuple(int(t) for t in rng.integers(1, 500, ln))
            for n, ln in (("A", 5), ("B", 3), ("C", 4), ("M", 6), ("T", 3), ("P0", 6),
                          ("P1", 2), ("P2", 9))}
    segs = {n: Segment(toks[n], SegmentKind.PRIVATE_HISTORY if n.startswith("P") else
                       SegmentKind.ROUND_TASK if n == "T" else SegmentKind.SHARED_OUTPUT)
            for n in toks}
    # entries: name -> (segment, first source position); A2 re-caches A later
    entries = [("A1", "A", 10), ("B", "B", 0), ("C", "C", 40), ("A2", "A", 3)]
    prompts = [["P0", "A", "T", "M", "B"], ["P1", "B", "A", "C", "A"], ["P2"]]
    return toks, segs, entries, prompts


def gen_prepare():
    """The reference's prepare_request on _prepare_world's prompts, plus the
    index's recency order afterwards and the entries an over-budget insert
    then evicts (lookups refresh recency in prompt/segment order)."""
    from roundkv.core import PromptLayout
    toks, segs, entries, prompts = _prepare_world()
    model = ModelConfig(num_layers=1, num_heads=1, head_dim=2, vocab_size=512)
    index = SegmentIndex(budget_bytes=10_000)
    name_of = {}
    for name, seg, src in entries:
        n = len(toks[seg])
        kv = LayeredKv(np.zeros((1, n, 1, 2), np.float32), np.zeros((1, n, 1, 2), np.float32),
                       np.arange(src, src + n))
        e = SegmentCacheEntry(segs[seg].digest, kv.positions, SimpleNamespace(kv=kv), b"ctx",
                              1000)
        index.insert(e)
        name_of[e.entry_id] = name
    out = {"prompts": prompts, "tokens": {n: list(t) for n, t in toks.items()},
           "entries": [list(e) for e in entries], "separator": model.separator_token,
           "requests": []}
    for i, names in enumerate(prompts):
        lay = PromptLayout(i, tuple(segs[n] for n in names))
        prep = prepare_request(lay, model, index, request_id=i)
        out["requests"].append({
            "tokens": prep.tokens.tolist(), "private_idx": prep.private_idx.tolist(),
            "structural_idx": prep.structural_idx.tolist(),
            "label_entry": [name_of.get(int(e), None) for e in prep.label_entry],
            "label_offset": prep.label_offset.tolist(),
            "hits": [[name_of[h.entry.entry_id], h.target_idx.tolist(), h.delta.tolist()]
                     for h in prep.hits]})
    out["recency"] = [name_of[e.entry_id] for e in index.entries()]
    evicted = []
    index._on_evict = lambda e: evicted.append(name_of[e.entry_id])
    n = len(toks["A"])
    kv = LayeredKv(np.zeros((1, n, 1, 2), np.float32), np.zeros((1, n, 1, 2), np.float32),
                   np.arange(n))
    index.insert(SegmentCacheEntry(b"x" * 16, kv.positions, SimpleNamespace(kv=kv), b"ctx", 7000))
    out["evicted_after_insert"] = evicted
    # errors
    bad = PromptLayout(9, (segs["P0"], segs["A"]))
    try:
        prepare_request(bad, ModelConfig(vocab_size=toks["A"][0] + 1), index)
    except ValueError as e:
        out["separator_error"] = str(e)
    return out


def main():
    golden = {
        "prepare": gen_prepare(),
        "t3": gen_t3(),
        "recovery": gen_recovery(),
        "toymodel": gen_toymodel(),
        "generator": "tests/golden/make_golden.py",
        "reference": "roundkv 0.1.0 (/root/reference/pkg/src)",
        "numpy": np.__version__,
        "rope": gen_rope(),
        "collector": gen_collector(),
        "family": gen_family(),
        "codec_trials": gen_codec_trials(),
        "known": gen_known_answers(),
        "restores": gen_restores(),
        "allocator": gen_allocator(),
        "segment_index": gen_segment_index(),
    }
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(golden, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    if sys.argv[1:] in (["--known-only"], ["--t3-only"], ["--prepare-only"]):  # one section
        path = os.path.join(HERE, "golden.json")
        with open(path) as f:
            golden = json.load(f)
        if sys.argv[1] == "--known-only":
            golden["known"] = gen_known_answers()
        elif sys.argv[1] == "--prepare-only":
            golden["prepare"] = gen_prepare()
        else:
            golden["t3"] = gen_t3()
        with open(path, "w") as f:
            json.dump(golden, f, indent=1, sort_keys=True)
        print("updated", sys.argv[1][2:], "in", path)
    else:
        main()
