"""Family restore (tdkv_restore_family: K1 with a diff overlay) against the
CPU oracle and against the per-mirror K3 decoder.

``fused_restore_many`` over mirrors that share masters runs the collector
kernel with each master as a source and each mirror as a job: a master tile
is staged once and written, rotated by the mirror's delta, to every mirror's
pool slots, except where the mirror's diff stores the (layer, block) -- then
the payload rows are rotated instead (the overlay precedes rotation,
restore.py:5-8).  Checked here:

* float32: bit-exact against ``oracle.fused_restore`` (K rotated in float64
  exactly as numpy, V a copy), over 18 families (two launches of <= 16
  masters), host and device masters, constant and per-token shifts;
* a diff whose V index list differs from K's (the TDDF escape form,
  diffstore.py:223-232) -- separate K and V overlay maps;
* bf16: bit-identical to the K3 form (same rotation arithmetic) and within
  the bf16 tolerance of the oracle;
* tiles never straddle a diff block (block sizes 8, 16, 32 with 2 KiB rows).
"""
import numpy as np
import pytest
import torch

import paper_2604_03143_b200 as tk
from paper_2604_03143_b200 import restore as rs
from oracle import roundkv_port as ref

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module", autouse=True)
def _built():
    tk.build_library()
    assert torch.cuda.is_available()


@pytest.fixture(autouse=True)
def _family_form(monkeypatch):
    """Small test families take the family-restore form too (by default
    fused_restore_many takes it from 32 mirrors per master)."""
    monkeypatch.setattr(rs, "_FAMILY_MIN", 1)


def _family_host(rng, L, T, H, D, n_mirrors, bs, frac=0.2):
    mk = rng.standard_normal((L, T, H, D)).astype(np.float32)
    mv = rng.standard_normal((L, T, H, D)).astype(np.float32)
    nb = -(-T // bs)
    mirrors, hints = [], []
    for _ in range(n_mirrors):
        k, v = mk.copy(), mv.copy()
        blocks = np.sort(rng.choice(nb, max(1, int(frac * nb)), replace=False))
        for b in blocks:
            lo, hi = b * bs, min(T, (b + 1) * bs)
            k[:, lo:hi] = rng.standard_normal(k[:, lo:hi].shape)
            v[:, lo:hi] = rng.standard_normal(v[:, lo:hi].shape)
        mirrors.append((k, v))
        hints.append(np.concatenate([np.arange(b * bs, min(T, (b + 1) * bs)) for b in blocks]))
    return mk, mv, mirrors, hints


def _pool_f32(cap, L, H, D):
    pool = tk.PagedPool(cap, L, H, D, device=DEV)
    junk = [pool.allocate(37 + 5 * i, 5000 + i) for i in range(6)]
    for j in junk[::2]:
        pool.free(j)
    return pool


def _oracle_pool(mk, mv, layers, bs, span, slots, cap):
    L, T, H, D = mk.shape
    wk = np.zeros((L, cap, H, D), np.float32)
    wv = np.zeros_like(wk)
    ref.fused_restore(mk, mv, layers, bs, span.old_positions, span.new_positions, slots, wk, wv,
                      10000.0)
    return wk[:, slots], wv[:, slots]


def _read(pool, smap):
    L = pool.num_layers
    k = np.stack([pool.read_rows(smap, layer)[0] for layer in range(L)]).astype(np.float32)
    v = np.stack([pool.read_rows(smap, layer)[1] for layer in range(L)]).astype(np.float32)
    return k, v


@pytest.mark.parametrize("bs", [8, 16, 32])
def test_family_restore_f32_bit_exact_many_families(bs):
    L, T, H, D = 2, 150, 4, 128              # 2 KiB rows: 8-row tiles inside every block
    rng = np.random.default_rng(bs)
    n_fam, per = 18, 2
    pos = np.arange(T, dtype=np.int64)
    handles, spans, want, fams = [], [], [], []
    for f in range(n_fam):
        mk, mv, mirrors, hints = _family_host(rng, L, T, H, D, per, bs)
        # half the families keep their master on the device (used in place)
        kv = (tk.LayeredKv(torch.from_numpy(mk).to(DEV), torch.from_numpy(mv).to(DEV), pos)
              if f % 2 else tk.LayeredKv(mk, mv, pos))
        entry = tk.MasterEntry(f, kv, pin_count=per)
        fams.append(entry)
        for i, (k, v) in enumerate(mirrors):
            diff = tk.encode_diff(tk.LayeredKv(mk, mv, pos), tk.LayeredKv(k, v, pos), hints[i],
                                  tk.CacheBlockConfig(bs))
            handles.append(tk.MirrorHandle(f, i + 1, entry, diff))
            if (f + i) % 3 == 0:             # a per-token shift
                new = np.cumsum(rng.integers(1, 5, T)).astype(np.int64) + 3
                spans.append(tk.PositionSpan(pos, new))
            else:
                spans.append(tk.PositionSpan.shifted(pos, int(rng.integers(-300, 5000))))
            want.append((mk, mv, ref.encode_diff(mk, mv, k, v, hints[i], bs)))
    pool = _pool_f32(2 * len(handles) * T + 512, L, H, D)
    maps = [pool.allocate(T, 100 + i) for i in range(len(handles))]
    before = tk.launch_count()
    tk.fused_restore_many(handles, spans, pool, maps, 10000.0)
    torch.cuda.synchronize()
    # two restore calls of <= 16 masters: K0 + K1 + the overlay pass each
    assert tk.launch_count() - before <= 6
    for i, (h, sp, smap) in enumerate(zip(handles, spans, maps)):
        mk, mv, layers = want[i]
        wk, wv = _oracle_pool(mk, mv, layers, bs, sp, smap.slots, pool.capacity)
        gk, gv = _read(pool, smap)
        assert np.array_equal(gv, wv), f"mirror {i}: V"
        assert np.array_equal(gk, wk), f"mirror {i}: K max err {np.abs(gk - wk).max()}"


def test_family_restore_separate_v_indices_f32():
    """The escape form: V changed in other blocks than K (separate index
    lists) -- the overlay maps K and V independently."""
    L, T, H, D, bs = 2, 96, 4, 128, 32
    rng = np.random.default_rng(7)
    mk = rng.standard_normal((L, T, H, D)).astype(np.float32)
    mv = rng.standard_normal((L, T, H, D)).astype(np.float32)
    pos = np.arange(T, dtype=np.int64)
    entry = tk.MasterEntry(0, tk.LayeredKv(mk, mv, pos), pin_count=3)
    handles, want = [], []
    for m in range(3):
        layers, rlayers = [], []
        for layer in range(L):
            ki = np.array([m % 3], np.int64)
            vi = np.array([(m + 1) % 3, 2], np.int64) if m != 2 else np.array([0, 2], np.int64)
            vi = np.unique(vi)
            kb = rng.standard_normal((ki.size, bs, H, D)).astype(np.float32)
            vb = rng.standard_normal((vi.size, bs, H, D)).astype(np.float32)
            layers.append(tk.LayerDiff(ki, kb, vb, v_indices=vi))
            rlayers.append(ref.DiffLayer(ki, kb, vb, v_indices=vi))
        diff = tk.BlockSparseDiff(L, bs, H, D, T, layers)
        handles.append(tk.MirrorHandle(0, m + 1, entry, diff))
        want.append(rlayers)
    spans = [tk.PositionSpan.shifted(pos, d) for d in (5, -7, 1000)]
    pool = _pool_f32(8 * T, L, H, D)
    maps = [pool.allocate(T, 10 + i) for i in range(3)]
    tk.fused_restore_many(handles, spans, pool, maps, 10000.0)
    torch.cuda.synchronize()
    for i in range(3):
        wk, wv = _oracle_pool(mk, mv, want[i], bs, spans[i], maps[i].slots, pool.capacity)
        gk, gv = _read(pool, maps[i])
        assert np.array_equal(gv, wv) and np.array_equal(gk, wk), f"mirror {i}"


def test_family_restore_bf16_equals_k3_and_oracle(monkeypatch):
    L, T, H, D, bs = 3, 700, 8, 128, 32
    rng = np.random.default_rng(11)
    mk, mv, mirrors, hints = _family_host(rng, L, T, H, D, 9, bs, 0.15)
    mkb = torch.from_numpy(mk).to(DEV).bfloat16()
    mvb = torch.from_numpy(mv).to(DEV).bfloat16()
    pos = np.arange(T, dtype=np.int64)
    master = tk.LayeredKv(mkb, mvb, pos)
    mir = [tk.LayeredKv(torch.from_numpy(k).to(DEV).bfloat16(),
                        torch.from_numpy(v).to(DEV).bfloat16(), pos) for k, v in mirrors]
    diffs = tk.encode_batch(master, mir, hints, tk.CacheBlockConfig(bs))
    entry = tk.MasterEntry(0, master, pin_count=len(diffs))
    handles = [tk.MirrorHandle(0, i + 1, entry, d) for i, d in enumerate(diffs)]
    spans = [tk.PositionSpan.shifted(pos, int(d)) for d in rng.integers(-500, 9000, len(diffs))]
    spans[3] = tk.PositionSpan(pos, np.cumsum(rng.integers(1, 3, T)).astype(np.int64))
    pool = tk.PagedPool(3 * len(diffs) * T + 256, L, H, D, dtype=torch.bfloat16, device=DEV)
    maps_fam = [pool.allocate(T, 10 + i) for i in range(len(diffs))]
    maps_k3 = [pool.allocate(T, 100 + i) for i in range(len(diffs))]
    tk.fused_restore_many(handles, spans, pool, maps_fam, 10000.0)
    monkeypatch.setattr(rs, "_FAMILY_K1", False)
    tk.fused_restore_many(handles, spans, pool, maps_k3, 10000.0)
    torch.cuda.synchronize()
    mk32, mv32 = mkb.float().cpu().numpy(), mvb.float().cpu().numpy()
    for i in range(len(diffs)):
        a = torch.from_numpy(maps_fam[i].slots).to(DEV)
        b = torch.from_numpy(maps_k3[i].slots).to(DEV)
        assert torch.equal(pool.k[:, a], pool.k[:, b]), f"mirror {i}: K differs from K3"
        assert torch.equal(pool.v[:, a], pool.v[:, b]), f"mirror {i}: V differs from K3"
        k32 = mir[i].k.float().cpu().numpy()
        v32 = mir[i].v.float().cpu().numpy()
        layers = ref.encode_diff(mk32, mv32, k32, v32, hints[i], bs)
        wk, wv = _oracle_pool(mk32, mv32, layers, bs, spans[i], maps_fam[i].slots, pool.capacity)
        gk, gv = _read(pool, maps_fam[i])
        assert np.array_equal(gv, wv)
        err = float((np.abs(gk - wk) / np.maximum(1.0, np.abs(wk))).max())
        assert err <= 1e-2, f"mirror {i}: K err {err}"


def test_family_restore_ledger_and_marks_match_k3(monkeypatch):
    """The ledger laws and pool bookkeeping do not depend on the kernel."""
    L, T, H, D, bs = 2, 64, 4, 128, 32
    rng = np.random.default_rng(3)
    mk, mv, mirrors, hints = _family_host(rng, L, T, H, D, 3, bs)
    pos = np.arange(T, dtype=np.int64)
    entry = tk.MasterEntry(0, tk.LayeredKv(mk, mv, pos), pin_count=3)
    handles = [tk.MirrorHandle(0, i + 1, entry,
                               tk.encode_diff(entry.kv, tk.LayeredKv(k, v, pos), h,
                                              tk.CacheBlockConfig(bs)))
               for i, ((k, v), h) in enumerate(zip(mirrors, hints))]
    spans = [tk.PositionSpan.shifted(pos, 9)] * 3
    got = []
    for fam in (True, False):
        monkeypatch.setattr(rs, "_FAMILY_K1", fam)
        pool = _pool_f32(6 * T, L, H, D)
        maps = [pool.allocate(T, i) for i in range(3)]
        led = tk.CostLedger(L)
        tk.fused_restore_many(handles, spans, pool, maps, 10000.0, ledger=led)
        torch.cuda.synchronize()
        got.append((led.as_dict(), [_read(pool, m) for m in maps]))
    assert got[0][0] == got[1][0]
    for (ka, va), (kb, vb) in zip(got[0][1], got[1][1]):
        assert np.array_equal(ka, kb) and np.array_equal(va, vb)


def test_k3_batch_of_host_masters_keeps_every_master(monkeypatch):
    """The per-mirror K3 form over mirrors of several HOST masters (fewer
    than _FAMILY_MIN mirrors per master): each master is uploaded once and
    stays alive until the launch -- descriptors hold raw addresses, so a
    master's device copy freed and reused by the next master's upload before
    the kernel ran would restore the wrong master (families interleaved
    A, B, A, C, B, ... to make every alias visible)."""
    monkeypatch.setattr(rs, "_FAMILY_K1", False)
    L, T, H, D, bs = 2, 96, 4, 128, 16
    rng = np.random.default_rng(11)
    fams = []
    for f in range(3):
        mk, mv, mirrors, hints = _family_host(rng, L, T, H, D, 2, bs)
        pos = np.arange(T, dtype=np.int64)
        entry = tk.MasterEntry(f, tk.LayeredKv(mk, mv, pos), pin_count=2)
        for (k, v), h in zip(mirrors, hints):
            d = tk.encode_diff(entry.kv, tk.LayeredKv(k, v, pos), h, tk.CacheBlockConfig(bs))
            fams.append((entry, d, k, v))
    order = [0, 2, 4, 1, 3, 5]              # families 0, 1, 2, 0, 1, 2
    handles = [tk.MirrorHandle(fams[i][0].family_id, 10 + i, fams[i][0], fams[i][1])
               for i in order]
    pool = _pool_f32(8 * T, L, H, D)
    maps = [pool.allocate(T, i) for i in range(len(order))]
    spans = [tk.PositionSpan.shifted(np.arange(T, dtype=np.int64), 5 + j)
             for j in range(len(order))]
    tk.fused_restore_many(handles, spans, pool, maps, 10000.0)
    torch.cuda.synchronize()
    for j, i in enumerate(order):
        _, _, k, v = fams[i]
        gk, gv = _read(pool, maps[j])
        assert np.array_equal(gv, v), f"mirror {j}: V"
        want = np.stack([ref.rope_apply(k[layer], np.full(T, 5 + j)) for layer in range(L)])
        assert np.array_equal(gk, want), f"mirror {j}: K"


def test_k3_batch_shared_shift_rows_match_oracle(monkeypatch):
    """The K3 form gives mirrors restored by the same constant shift one
    shared cos/sin row (a repeated shift -> the cached one-row table): a batch
    mixing repeated shifts, a zero shift, a negative shift and a per-token
    shift restores every mirror bit-exactly as the oracle (float32)."""
    monkeypatch.setattr(rs, "_FAMILY_K1", False)
    L, T, H, D, bs = 2, 80, 2, 64, 16
    rng = np.random.default_rng(29)
    mk, mv, mirrors, hints = _family_host(rng, L, T, H, D, 7, bs)
    pos = np.arange(T, dtype=np.int64)
    entry = tk.MasterEntry(0, tk.LayeredKv(mk, mv, pos), pin_count=7)
    diffs = [tk.encode_diff(entry.kv, tk.LayeredKv(k, v, pos), h, tk.CacheBlockConfig(bs))
             for (k, v), h in zip(mirrors, hints)]
    handles = [tk.MirrorHandle(0, 1 + i, entry, d) for i, d in enumerate(diffs)]
    per_token = np.cumsum(rng.integers(1, 5, T)).astype(np.int64) + 3
    spans = [tk.PositionSpan.shifted(pos, 16), tk.PositionSpan.shifted(pos, 16),
             tk.PositionSpan.shifted(pos, 0), tk.PositionSpan(pos, per_token),
             tk.PositionSpan.shifted(pos, -9), tk.PositionSpan.shifted(pos, 16),
             tk.PositionSpan.shifted(pos, -9)]
    pool = _pool_f32(8 * T + 512, L, H, D)
    maps = [pool.allocate(T, 100 + i) for i in range(len(handles))]
    tk.fused_restore_many(handles, spans, pool, maps, 10000.0)
    torch.cuda.synchronize()
    for j, (span, smap) in enumerate(zip(spans, maps)):
        k, v = mirrors[j]
        layers = ref.encode_diff(mk, mv, k, v, hints[j], bs)
        wk, wv = _oracle_pool(mk, mv, layers, bs, span, smap.slots, pool.capacity)
        gk, gv = _read(pool, smap)
        assert np.array_equal(gv, wv), f"mirror {j}: V"
        assert np.array_equal(gk, wk), f"mirror {j}: K"
