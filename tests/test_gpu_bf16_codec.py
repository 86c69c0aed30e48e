"""bf16 codec parity: the kernels the bench times (K2 ``diff_encode_kernel``
on bf16 planes, K3 ``rows_tma_kernel`` on bf16 pools) against the CPU oracle
run on the float32-upcast inputs.

The reference is float32-only (core.py:180-181); a bf16 cache upcasts to
float32 exactly, so for the encoder everything is bit-exact against
``oracle.encode_diff`` on the upcast planes: the change masks (float '!='
semantics, +0 == -0, NaN != NaN -- diffstore.py:151-153), the ascending index
lists (diffstore.py:166-173), the zero-padded payload bytes (upcast), the
first soundness violation and its message (diffstore.py:156-164), and the
float32 TDDF wire image (diffstore.py:210-239).  Restores rotate bf16 in
float32 and round once to bf16, so rotated K is held to the north_star bf16
tolerance -- max |got - want| / max(1, |want|) <= 1e-2 against
``oracle.fused_restore`` -- and V (a copy) is bit-exact.

Shapes: slices of configs C2 (L=28 -> fewer layers, H=4, D=128, T=4,624,
nb=145 with a 16-row last block) and C4 (T=12,320, nb=385), families of 8 to
49 mirrors (the bench encodes 49 mirrors of one master in one launch, so the
look-back compaction runs across many pairs).
"""
import numpy as np
import pytest
import torch

import paper_2604_03143_b200 as tk
from oracle import roundkv_port as ref

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)
BF16_TOL = 1e-2
BS = 32


@pytest.fixture(scope="module", autouse=True)
def _built():
    tk.build_library()
    assert torch.cuda.is_available()


def _up(x: torch.Tensor) -> np.ndarray:
    """bf16 device plane -> float32 host (exact)."""
    return x.float().cpu().numpy()


def _bf16_close(got: np.ndarray, want: np.ndarray) -> float:
    return float((np.abs(got - want) / np.maximum(1.0, np.abs(want))).max()) if got.size else 0.0


def _family(seed, L, T, H, D, n_mirrors, frac):
    """Master + mirrors in bf16 on the device: each mirror re-draws a random
    ``frac`` of its blocks in every layer (the perturb_blocks recipe,
    conftest.py:63-73), hints = those blocks plus one hinted-but-identical
    block.  Edge cases are planted in the first mirrors:
      m0: -0.0 where the master has +0.0 in an UNHINTED block (unchanged),
      m1: a block changed in V only,
      m2: NaN in both master and mirror at the same element of a hinted
          block (NaN != NaN: stored),
      m3: the last (partial, T % 32 rows) block re-drawn,
      m4: every block hinted, nothing re-drawn (only the shared-NaN block
          is stored)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    nb = -(-T // BS)
    mk = torch.randn((L, T, H, D), generator=g).to(torch.bfloat16)
    mv = torch.randn((L, T, H, D), generator=g).to(torch.bfloat16)
    mk[0, 5, 0, 3] = 0.0                    # a +0 for m0's signed-zero flip
    rng = np.random.default_rng(seed)
    # a NaN shared by master and every mirror at (layer 1, token 70): block 2
    # differs from itself (NaN != NaN) in every mirror, so it is hinted in all
    mk[1 % L, 70, 0, 0] = float("nan")
    mirrors, hints = [], []
    for m in range(n_mirrors):
        k, v = mk.clone(), mv.clone()
        nchg = max(1, int(frac * nb))
        blocks = sorted(rng.choice(nb, nchg, replace=False).tolist())
        if m == 3 and nb - 1 not in blocks:
            blocks.append(nb - 1)
        if m == 4:
            blocks = []
        if m == 0:
            blocks = [b for b in blocks if b != 0]
        for b in blocks:
            lo, hi = b * BS, min(T, b * BS + BS)
            k[:, lo:hi] = torch.randn((L, hi - lo, H, D), generator=g).to(torch.bfloat16)
            v[:, lo:hi] = torch.randn((L, hi - lo, H, D), generator=g).to(torch.bfloat16)
        hinted = set(blocks) | {2}
        if m == 0:
            k[0, 5, 0, 3] = -0.0                            # block 0, unhinted
        if m == 1:
            free = [b for b in range(nb) if b not in hinted]
            b = free[len(free) // 2]
            v[L - 1, b * BS + 3, H - 1, D - 1] += 1.0       # V-only change, hinted below
            hinted.add(b)
        if m == 2:
            b = [x for x in range(nb) if x not in hinted][0]
            k[0, b * BS + 1, 1, 2] = float("nan")
            mk_b = mk[0, b * BS + 1, 1, 2]
            hinted.add(b)
            assert mk_b == mk_b                              # master side is a number
        if m == 4:
            hinted = set(range(nb))
        hint_pos = np.concatenate([np.arange(b * BS, min(T, b * BS + BS)) for b in sorted(hinted)])
        mirrors.append((k, v))
        hints.append(hint_pos.astype(np.int64))
    return mk, mv, mirrors, hints


def _layered(k, v, T):
    return tk.LayeredKv(k.to(DEV), v.to(DEV), np.arange(T, dtype=np.int64))


@pytest.mark.parametrize("L,T,n_mirrors,frac", [
    (4, 4624, 8, 0.1),         # C2 slice (nb = 145, partial last block)
    (2, 4624, 49, 0.1),        # the bench's 49-mirror family at C2's T
    (2, 12320, 8, 0.5),        # C4 slice: nb = 385, AgentSociety-like churn
    (28, 4624, 8, 0.05),       # C2 full depth
])
def test_encode_batch_bf16_bit_exact_against_oracle(L, T, n_mirrors, frac):
    H, D = 4, 128
    mk, mv, mirrors, hints = _family(1000 + L + n_mirrors, L, T, H, D, n_mirrors, frac)
    master = _layered(mk, mv, T)
    mir_kv = [_layered(k, v, T) for k, v in mirrors]
    diffs = tk.encode_batch(master, mir_kv, hints, tk.CacheBlockConfig(BS))
    assert len(diffs) == n_mirrors
    mk32, mv32 = mk.float().numpy(), mv.float().numpy()
    stored_total = 0
    for i, ((k, v), h, diff) in enumerate(zip(mirrors, hints, diffs)):
        want = ref.encode_diff(mk32, mv32, k.float().numpy(), v.float().numpy(), h, BS)
        got_idx = [ld.indices.tolist() for ld in diff.layers]
        assert got_idx == [w.indices.tolist() for w in want], f"mirror {i}: index lists"
        for layer, (ld, w) in enumerate(zip(diff.layers, want)):
            assert np.array_equal(_up(ld.k_blocks).view(np.uint32), w.k_blocks.view(np.uint32)), \
                (i, layer)
            assert np.array_equal(_up(ld.v_blocks).view(np.uint32), w.v_blocks.view(np.uint32)), \
                (i, layer)
        # the float32 TDDF image (GPU-packed, bf16 -> f32 on the fly) equals
        # the oracle's serialization byte for byte
        wire = tk.serialize_diff(diff)
        assert wire == ref.serialize(want, BS, H, D, T), f"mirror {i}: wire bytes"
        assert len(wire) == tk.wire_nbytes(diff)
        stored_total += sum(diff.changed_blocks_per_layer)
    # the planted cases behaved as the reference semantics say
    assert 0 not in diffs[0].layers[0].indices.tolist()            # -0 == +0
    # m4: every block hinted, only the shared-NaN block differs (from itself)
    assert [ld.indices.tolist() for ld in diffs[4].layers] == \
        [[2] if layer == 1 % L else [] for layer in range(L)]
    assert 2 in diffs[min(5, n_mirrors - 1)].layers[1 % L].indices.tolist()  # NaN != NaN
    assert stored_total > 0


def test_encode_batch_bf16_first_violation_in_list_order():
    """Two mirrors violate their hints; the error names the first mirror in
    list order at its first (layer, block) in layer-major order, with the
    reference's max-abs message computed on the upcast planes."""
    L, T, H, D = 3, 4624, 4, 128
    mk, mv, mirrors, hints = _family(77, L, T, H, D, 8, 0.1)
    nb = -(-T // BS)
    hinted5 = set((hints[5] // BS).tolist())
    hinted6 = set((hints[6] // BS).tolist())
    b5 = [b for b in range(nb) if b not in hinted5][7]
    b6 = [b for b in range(nb) if b not in hinted6][0]
    k5, v5 = mirrors[5]
    v5[2, b5 * BS + 4, 1, 9] += 3.0                  # layer 2
    k5[1, b5 * BS + 9, 0, 0] += 0.25                 # layer 1: the first in layer-major order
    k6, _ = mirrors[6]
    k6[0, b6 * BS, 0, 0] += 1.0
    master = _layered(mk, mv, T)
    with pytest.raises(tk.HintSoundnessError) as err:
        tk.encode_batch(master, [_layered(k, v, T) for k, v in mirrors], hints,
                        tk.CacheBlockConfig(BS))
    with pytest.raises(ref.HintViolation) as want:
        ref.encode_diff(mk.float().numpy(), mv.float().numpy(), k5.float().numpy(),
                        v5.float().numpy(), hints[5], BS)
    assert str(err.value) == str(want.value)
    assert f"layer 1 block {b5}" in str(err.value)


def _pool_with_holes(n_tokens, L, H, D, seed):
    """A bf16 pool whose free list is fragmented (slot maps are not runs)."""
    pool = tk.PagedPool(n_tokens, L, H, D, dtype=torch.bfloat16, device=DEV)
    rng = np.random.default_rng(seed)
    junk = [pool.allocate(int(rng.integers(5, 70)), 1000 + i) for i in range(12)]
    for j in junk[::2]:
        pool.free(j)
    return pool


@pytest.mark.parametrize("T,deltas", [
    (4624, [0, 16, -5, 7000]),
    (700, [3, -700 + 1, 123456, 1]),
])
def test_fused_restore_bf16_against_oracle(T, deltas):
    """fused_restore (one mirror per call) and fused_restore_many (the
    batched family form the bench times) on bf16 pools, several constant
    shifts and one per-token shift, fragmented slot maps."""
    L, H, D = 3, 4, 128
    n = len(deltas) + 1
    mk, mv, mirrors, hints = _family(31 + T, L, T, H, D, n, 0.2)
    mk[1 % L, 70, 0, 0] = 0.5                        # finite planes for the restore check
    for k, _ in mirrors:
        k[1 % L, 70, 0, 0] = 0.5
        k.nan_to_num_(0.0)
    master = _layered(mk, mv, T)
    diffs = tk.encode_batch(master, [_layered(k, v, T) for k, v in mirrors], hints,
                            tk.CacheBlockConfig(BS))
    entry = tk.MasterEntry(0, master, pin_count=n)
    handles = [tk.MirrorHandle(0, i + 1, entry, d) for i, d in enumerate(diffs)]
    pos = np.arange(T, dtype=np.int64)
    rng = np.random.default_rng(T)
    spans = [tk.PositionSpan.shifted(pos, d) for d in deltas]
    # per-token shift: strictly increasing new positions with varying gaps
    new = np.cumsum(rng.integers(1, 4, T)).astype(np.int64) + 11
    spans.append(tk.PositionSpan(pos, new))
    pool = _pool_with_holes(2 * n * T + 4096, L, H, D, T)
    maps_one = [pool.allocate(T, 10 + i) for i in range(n)]
    maps_many = [pool.allocate(T, 100 + i) for i in range(n)]
    for h, sp, m in zip(handles, spans, maps_one):
        tk.fused_restore(h, sp, pool, m, 10000.0)
    tk.fused_restore_many(handles, spans, pool, maps_many, 10000.0)
    torch.cuda.synchronize()
    mk32, mv32 = mk.float().numpy(), mv.float().numpy()
    cap = pool.capacity
    worst = 0.0
    for i, ((k, v), h, sp) in enumerate(zip(mirrors, hints, spans)):
        layers = ref.encode_diff(mk32, mv32, k.float().numpy(), v.float().numpy(), h, BS)
        wk = np.zeros((L, cap, H, D), np.float32)
        wv = np.zeros_like(wk)
        slots = maps_one[i].slots
        ref.fused_restore(mk32, mv32, layers, BS, sp.old_positions, sp.new_positions, slots,
                          wk, wv, 10000.0)
        for smap in (maps_one[i], maps_many[i]):
            gk = np.stack([pool.read_rows(smap, l)[0] for l in range(L)]).astype(np.float32)
            gv = np.stack([pool.read_rows(smap, l)[1] for l in range(L)]).astype(np.float32)
            assert np.array_equal(gv, wv[:, slots]), f"mirror {i}: V"
            err = _bf16_close(gk, wk[:, slots])
            worst = max(worst, err)
            assert err <= BF16_TOL, f"mirror {i}: K err {err}"
        # the batched and the per-call forms run the same arithmetic
        a = torch.from_numpy(maps_one[i].slots).to(DEV)
        b = torch.from_numpy(maps_many[i].slots).to(DEV)
        assert torch.equal(pool.k[:, a], pool.k[:, b]) and torch.equal(pool.v[:, a], pool.v[:, b])
    print(f"bf16 restore worst relative K error vs oracle: {worst:.2e}")


def test_read_rows_returns_bf16_as_host_arrays():
    pool = tk.PagedPool(64, 2, 4, 128, dtype=torch.bfloat16, device=DEV)
    m = pool.allocate(10, 0)
    pool.write_rows(m, 1, np.ones((10, 4, 128), np.float32), np.zeros((10, 4, 128), np.float32))
    k, v = pool.read_rows(m, 1)
    assert isinstance(k, np.ndarray) and (k == 1).all() and (v == 0).all()
    kd, _ = pool.read_rows_device(m, 1)
    assert kd.is_cuda and kd.dtype == torch.bfloat16


def test_restore_and_pool_reject_mismatched_geometry():
    """Descriptors are built from raw pointers: every geometry mismatch is a
    ValueError / IndexError before any launch, as numpy raises in the
    reference (restore.py:68-99, paged_pool.py:150-164)."""
    T, L, H, D = 96, 2, 4, 128
    mk, mv, mirrors, hints = _family(5, L, T, H, D, 5, 0.3)
    mk.nan_to_num_(0.0)
    for k, _ in mirrors:
        k.nan_to_num_(0.0)
    master = _layered(mk, mv, T)
    diffs = tk.encode_batch(master, [_layered(k, v, T) for k, v in mirrors], hints,
                            tk.CacheBlockConfig(BS))
    entry = tk.MasterEntry(0, master, pin_count=1)
    h = tk.MirrorHandle(0, 1, entry, diffs[1])
    span = tk.PositionSpan.shifted(np.arange(T), 3)
    small = tk.PagedPool(T + 8, L, H, D, dtype=torch.bfloat16, device=DEV)
    big = tk.PagedPool(4 * T, L, H, D, dtype=torch.bfloat16, device=DEV)
    big.allocate(2 * T, 0)
    far = big.allocate(T, 1)                       # slots beyond small's capacity
    with pytest.raises(IndexError):
        tk.fused_restore(h, span, small, far, 10000.0)
    with pytest.raises(IndexError):
        tk.fused_restore_many([h], [span], small, [far], 10000.0)
    with pytest.raises(IndexError):
        tk.dense_restore(h, span, small, far, 10000.0)
    with pytest.raises(IndexError):
        small.write_rows(far, 0, np.zeros((T, H, D), np.float32), np.zeros((T, H, D), np.float32))
    wrong_heads = tk.PagedPool(4 * T, L, H // 2, D, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(ValueError, match="do not match the pool"):
        tk.fused_restore(h, span, wrong_heads, wrong_heads.allocate(T, 2), 10000.0)
    other = tk.LayeredKv(mk[:1].clone().to(DEV), mv[:1].clone().to(DEV), np.arange(T))
    bad = tk.MirrorHandle(0, 2, tk.MasterEntry(1, other, pin_count=1), diffs[1])
    one_layer = tk.PagedPool(4 * T, 1, H, D, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(ValueError, match="diff does not describe"):
        tk.fused_restore(bad, span, one_layer, one_layer.allocate(T, 3), 10000.0)
    with pytest.raises(IndexError):
        small.read_rows(small.allocate(4, 9), L)
