"""The drop-in under the reference's own caller: trace._run_t3
(trace.py:332-403) -- prepare, group, collective_recover, _write_cache,
DiffStore.encode_family, _verify_family_restores (fused vs dense restore
bit-equality, trace.py:289-329), the remainder's serial recovery, the
fidelity and the ledger row -- replayed round by round with this repo's
functions in place of the reference's, against the report rows the
reference's own ``run_trace(spec, paths=("T3",))`` produced
(tests/golden/make_golden.py: gen_t3).

The control flow below restates _run_t3 / _verify_family_restores /
_finish_row line by line (each step cites its lines); the prepared requests
(prompt layout, hit resolution: host-side prepare_request, out of scope per
SURVEY §2) and the seeded segment rows are the reference's, recorded by
wrapping its own calls.  Every counter of the report row must match exactly:
rope calls, selection passes, recomputed tokens, bytes stored (dense / diff),
bytes moved, dense mirror allocations, pool peak occupancy, temp buffer peak,
the compression lists (families, payload and serialized bytes, ratios,
changed blocks), restores verified and pool exhaustion; the elected masters
and mirror hints are exact; the fidelity errors (K/V rows vs the full
prefill oracles) agree within 1e-6 absolute -- the recovered caches match the
reference's within 1e-5 (tests/test_gpu_pic.py).
"""
import numpy as np
import pytest

import paper_2604_03143_b200 as tk
from helpers import load_golden, load_npz
from oracle import roundkv_port as ref
from paper_2604_03143_b200 import pic
from paper_2604_03143_b200.rounds import ToyGroup, ToyHit, ToyRequest

pytestmark = pytest.mark.gpu
G = load_golden()["t3"]


class _Cfg:
    def __init__(self, L, H, D, V):
        self.num_layers, self.num_heads, self.head_dim, self.vocab_size = L, H, D, V
        self.rope_base = 10000.0


class _Weights:
    def __init__(self, L, H, D, V, seed):
        w = ref.build_weights(L, H, D, V, seed)
        self.config = _Cfg(L, H, D, V)
        self.embed, self.wq, self.wk, self.wv, self.wm = w.embed, w.wq, w.wk, w.wv, w.wm


class _Pic:
    recompute_fraction = 0.15
    check_layer = 1


def _host(x):
    return x if isinstance(x, np.ndarray) else x.detach().cpu().numpy()


def _prep(z, m, seed_masters):
    """The reference's PreparedRequest (pic.py:67-98) of one prompt: hits
    point at the seeded masters' caches (entry.kv_ref.kv, pic.py:139)."""
    tag = m["tag"]
    hits = [ToyHit(seed_masters[h["seed"]].kv, np.asarray(h["target"], np.int64))
            for h in m["hits"]]
    return ToyRequest(m["rid"], z[f"{tag}_tokens"], z[f"{tag}_positions"],
                      z[f"{tag}_private_idx"], z[f"{tag}_structural_idx"], hits,
                      z[f"{tag}_label_entry"], z[f"{tag}_label_offset"])


def _write_cache(pool, slot_map, kv):                       # trace.py:148-152
    if slot_map is None:
        return
    for layer in range(kv.num_layers):
        pool.write_rows(slot_map, layer, kv.k[layer], kv.v[layer])


def _fidelity(results, oracles):                            # trace.py:130-145
    k_all, v_all = [], []
    for got, (ok, ov) in zip(results, oracles):
        dk = _host(got.k) - ok
        dv = _host(got.v) - ov
        k_all.append(np.sqrt(np.einsum("lthd,lthd->lt", dk, dk)).ravel())
        v_all.append(np.sqrt(np.einsum("lthd,lthd->lt", dv, dv)).ravel())
    k, v = np.concatenate(k_all), np.concatenate(v_all)
    return {"mean_k_err": float(k.mean()), "max_k_err": float(k.max()),
            "mean_v_err": float(v.mean()), "max_v_err": float(v.max())}


def _verify_family_restores(pool, enc, ledger, row, L, shift, rope_base):  # trace.py:289-329
    for rid, handle in sorted(enc.mirrors.items()):
        total = handle.master.kv.num_tokens
        try:
            fused_map = pool.allocate(total, request_id=1_000_000 + rid)
        except tk.OutOfSlotsError:
            row["pool_exhausted"] = True
            return
        try:
            dense_map = pool.allocate(total, request_id=2_000_000 + rid)
        except tk.OutOfSlotsError:
            pool.free(fused_map)
            row["pool_exhausted"] = True
            return
        span = tk.PositionSpan.shifted(handle.positions, shift)
        tk.fused_restore(handle, span, pool, fused_map, rope_base, ledger=ledger)
        tk.dense_restore(handle, span, pool, dense_map, rope_base, ledger=tk.CostLedger(L))
        for layer in range(L):
            fk, fv = pool.read_rows(fused_map, layer)
            dk, dv = pool.read_rows(dense_map, layer)
            assert np.array_equal(fk, dk) and np.array_equal(fv, dv), (rid, layer)
        pool.free(fused_map)
        pool.free(dense_map)
        row["restores_verified"] += 1


@pytest.mark.parametrize("case", sorted(G))
def test_t3_rounds_reproduce_reference_report(case):
    meta = G[case]
    z = load_npz("t3.npz")
    L, H, D, V, seed = meta["model"]
    weights = _Weights(L, H, D, V, seed)
    blocks = tk.CacheBlockConfig(meta["block_size"])
    # one path state for all rounds (trace.py:117-127)
    pool = tk.PagedPool(meta["capacity"], L, H, D, block_size=meta["block_size"])
    store = tk.DiffStore(blocks)
    seed_masters = {}
    for rmeta in meta["rounds"]:
        want = rmeta["row"]
        pool.reset_peak()
        for key in rmeta["seeds"]:                          # _seed_path, trace.py:176-181
            rows = tk.LayeredKv(z[key + "_k"], z[key + "_v"], z[key + "_pos"])
            seed_masters[key] = store.register_dense(rows, tokens=z[key + "_tokens"].tolist())
        ledger = tk.CostLedger(L)
        row = {"hit_segments": 0, "restores_verified": 0, "pool_exhausted": False}
        # _prepare_round (trace.py:184-206): slots in prompt order; the
        # allocator must hand out the reference's slot maps
        maps = {}
        for agent, flat_len in rmeta["prompts"]:
            try:
                maps[agent] = pool.allocate(flat_len, request_id=agent)
            except tk.OutOfSlotsError:
                maps[agent] = None
                row["pool_exhausted"] = True
        groups = []
        for g in rmeta["groups"]:
            members = []
            for m in g["members"]:
                p = _prep(z, m, seed_masters)
                p.slot_map = maps[m["rid"]]
                assert (None if p.slot_map is None else p.slot_map.slots.tolist()) == m["slots"]
                members.append(p)
            groups.append((ToyGroup(members), g))
        remainder = []
        for m in rmeta["remainder"]:
            p = _prep(z, m, seed_masters)
            p.slot_map = maps[m["rid"]]
            remainder.append(p)
        row["hit_segments"] = sum(len(p.hits) for grp, _ in groups for p in grp.members) + \
            sum(len(p.hits) for p in remainder)
        results_by_id = {}
        compression = {"families": 0, "mirror_serialized_bytes": [], "mirror_payload_bytes": [],
                       "mirror_ratios": [], "changed_blocks": []}
        for group, gmeta in groups:                         # trace.py:365-386
            results, plan = pic.collective_recover(weights, group, _Pic, ledger)
            assert plan.master_id == gmeta["master_id"]
            assert {str(k): v.tolist() for k, v in plan.mirror_diff_hints.items()} == gmeta["hints"]
            for prep in group.members:
                result = results[prep.request_id]
                _write_cache(pool, prep.slot_map, result.kv)
                results_by_id[prep.request_id] = result
            master_prep = next(p for p in group.members if p.request_id == plan.master_id)
            enc = store.encode_family(plan, results, tokens=master_prep.tokens.tolist())
            stats = enc.stats
            ledger.record_stored(stats.dense_nbytes, sum(stats.diff_serialized_nbytes))
            compression["families"] += 1
            compression["mirror_serialized_bytes"] += stats.diff_serialized_nbytes
            compression["mirror_payload_bytes"] += stats.diff_payload_nbytes
            compression["mirror_ratios"] += [float(r) for r in stats.ratios]
            compression["changed_blocks"] += stats.changed_blocks
            _verify_family_restores(pool, enc, ledger, row, L, meta["restore_shift"], 10000.0)
        for prep in remainder:                              # trace.py:388-393
            result = pic.recover_prepared(weights, prep, _Pic, ledger)
            ledger.record_stored(result.kv.dense_nbytes, 0)
            store.register_dense(result.kv, tokens=prep.tokens.tolist())
            _write_cache(pool, prep.slot_map, result.kv)
            results_by_id[prep.request_id] = result
        ordered = [results_by_id[agent].kv for agent, _ in rmeta["prompts"]]
        oracles = [(z[f"{case}_oracle_r{rmeta['round']}_a{a}_k"],
                    z[f"{case}_oracle_r{rmeta['round']}_a{a}_v"])
                   for a in range(len(rmeta["prompts"]))]
        fid = _fidelity(ordered, oracles)
        ledger.pool_peak_occupancy = pool.peak_allocated    # _finish_row, trace.py:221-229
        counters = ledger.as_dict()
        dense = [kv.dense_nbytes for kv in ordered]
        storage = ledger.bytes_stored_total / (sum(dense) / len(dense))
        for m in maps.values():                             # _free_maps
            if m is not None:
                pool.free(m)

        assert len(groups) == want["num_groups"] and len(remainder) == want["num_remainder"]
        assert row["hit_segments"] == want["hit_segments"]
        assert row["restores_verified"] == want["restores_verified"]
        assert row["pool_exhausted"] == want["pool_exhausted"]
        for key, value in counters.items():
            assert value == want[key], (rmeta["round"], key, value, want[key])
        assert storage == want["storage_cost_dense_units"]
        assert compression == want["compression"], rmeta["round"]
        for key, value in fid.items():
            assert abs(value - want["fidelity"][key]) <= 1e-6, (key, value, want["fidelity"][key])
    pool.check_conservation()
