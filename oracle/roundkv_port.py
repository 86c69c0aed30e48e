"""CPU oracle for the TokenDance collector + diff-codec hot path.

TEST INFRASTRUCTURE ONLY.  This module is a plain-numpy restatement of the
reference package ``roundkv`` 0.1.0 (``/root/reference/pkg/src/roundkv``) for
the functions on the hot path.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it,
and only as the checker or the timed CPU baseline -- never as the product.
The product path (``paper_2604_03143_b200``) never imports this module.

Parity pinning: every function here is checked bit-for-bit against golden
vectors produced by the reference itself (``tests/golden/make_golden.py``
imports ``roundkv`` from ``/root/reference`` in the build container and
records its outputs under ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.

Arithmetic conventions restated from the reference:
  * rotary pairs are interleaved ``(2j, 2j+1)``; ``inv_freq = base^(-2j/D)``
    in float64; angle ``= delta * inv_freq`` in float64; the rotation is
    evaluated in float64 and rounded once to float32
    (``toymodel.py:60-83``);
  * a span whose deltas are all zero is an exact copy (``toymodel.py:86-96``,
    ``pic.py:228``);
  * diff block equality is float ``==`` (``np.array_equal``), so ``+0 == -0``
    and ``NaN != NaN`` (``diffstore.py:151-153``).
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "inv_freq", "rope_apply", "rope_apply_neox", "rope_recover", "block_count", "block_range",
    "valid_len", "allocate_slots", "CollectJob", "collect_into_contexts",
    "collect_into_pool", "DiffLayer", "HintViolation", "encode_diff",
    "decode_dense", "wire_size", "serialize", "deserialize", "WireError",
    "fused_restore", "dense_restore", "mirror_hints", "select_master",
]


# ---------------------------------------------------------------------------
# rotary arithmetic -- toymodel.py:60-96


def inv_freq(head_dim: int, base: float = 10000.0) -> np.ndarray:
    """``base ** (-(0,2,4,..)/D)`` in float64 (toymodel.py:74)."""
    exps = -np.arange(0, head_dim, 2, dtype=np.float64) / head_dim
    return float(base) ** exps


def rope_apply(k: np.ndarray, positions: np.ndarray, base: float = 10000.0) -> np.ndarray:
    """Rotate interleaved pairs of ``k`` (T, H, D) by ``positions`` (T,).

    Restates toymodel.py:60-83: float64 angles, float64 rotation, one final
    round-to-nearest cast to float32.
    """
    if k.ndim != 3:
        raise ValueError("expected (tokens, heads, head_dim)")
    t, _, d = k.shape
    if d % 2:
        raise ValueError("head_dim must be even")
    pos = np.asarray(positions, dtype=np.float64)
    if pos.shape != (t,):
        raise ValueError("one position per token required")
    theta = pos.reshape(t, 1) * inv_freq(d, base).reshape(1, d // 2)
    c = np.cos(theta).reshape(t, 1, d // 2)
    s = np.sin(theta).reshape(t, 1, d // 2)
    pairs = k.astype(np.float64).reshape(k.shape[0], k.shape[1], d // 2, 2)
    even, odd = pairs[..., 0], pairs[..., 1]
    out = np.stack((even * c - odd * s, even * s + odd * c), axis=-1)
    return out.reshape(k.shape).astype(np.float32)


def rope_apply_neox(k: np.ndarray, positions: np.ndarray, base: float = 10000.0) -> np.ndarray:
    """The rotate-half (GPT-NeoX / Llama) pairing of the same rotation: element
    j pairs with j + D/2 of its head, angle index j (an extension beyond the
    reference, which pairs interleaved elements, toymodel.py:78-82); the
    arithmetic is rope_apply's -- float64 angles and rotation, one cast to
    float32."""
    if k.ndim != 3:
        raise ValueError("expected (tokens, heads, head_dim)")
    t, _, d = k.shape
    if d % 2:
        raise ValueError("head_dim must be even")
    pos = np.asarray(positions, dtype=np.float64)
    if pos.shape != (t,):
        raise ValueError("one position per token required")
    theta = pos.reshape(t, 1) * inv_freq(d, base).reshape(1, d // 2)
    c = np.cos(theta).reshape(t, 1, d // 2)
    s = np.sin(theta).reshape(t, 1, d // 2)
    x = k.astype(np.float64)
    lo, hi = x[..., :d // 2], x[..., d // 2:]
    return np.concatenate((lo * c - hi * s, lo * s + hi * c), axis=-1).astype(np.float32)


def rope_recover(old_positions: np.ndarray, new_positions: np.ndarray,
                 k: np.ndarray, base: float = 10000.0) -> np.ndarray:
    """Re-encode K rows from old to new positions (toymodel.py:86-96)."""
    old = np.asarray(old_positions, dtype=np.int64)
    new = np.asarray(new_positions, dtype=np.int64)
    if k.shape[0] != old.size:
        raise ValueError("span length must match token count")
    delta = new - old
    if not delta.any():
        return k.copy()
    return rope_apply(k, delta, base)


# ---------------------------------------------------------------------------
# block geometry -- core.py:240-263


def block_count(num_tokens: int, block_size: int) -> int:
    return (num_tokens + block_size - 1) // block_size


def block_range(b: int, num_tokens: int, block_size: int) -> Tuple[int, int]:
    lo = b * block_size
    if lo >= num_tokens:
        raise ValueError("block index out of range")
    return lo, min(lo + block_size, num_tokens)


def valid_len(num_tokens: int, block_size: int) -> int:
    rem = num_tokens % block_size
    return rem if rem else min(block_size, num_tokens)


# ---------------------------------------------------------------------------
# slot allocation policy -- paged_pool.py:106-135


def allocate_slots(free: np.ndarray, num_tokens: int, block_size: int) -> np.ndarray:
    """Pick ``num_tokens`` slots from the boolean ``free`` mask (mutated).

    Policy restated from paged_pool.py:117-133: scan blocks in ascending
    order and take each block whose every slot is free (a prefix of it when
    less is needed); then top up with the lowest remaining free slots.
    """
    cap = free.size
    if num_tokens > int(free.sum()):
        raise RuntimeError(f"requested {num_tokens} slots, {int(free.sum())} free")
    picked: List[int] = []
    need = num_tokens
    for b in range(block_count(cap, block_size)):
        if need <= 0:
            break
        lo, hi = b * block_size, min(b * block_size + block_size, cap)
        if free[lo:hi].all():
            n = min(need, hi - lo)
            picked.extend(range(lo, lo + n))
            need -= n
    if need > 0:
        taken = np.zeros(cap, dtype=bool)
        taken[picked] = True
        rest = np.flatnonzero(free & ~taken)[:need]
        picked.extend(rest.tolist())
    out = np.asarray(picked, dtype=np.int64)
    free[out] = False
    return out


# ---------------------------------------------------------------------------
# the KV Collector -- pic.py:192-235 (+ paged_pool.py:150-156 for the pool)


@dataclass
class CollectJob:
    """One (agent, shared segment) hit.

    ``master_k``/``master_v``: (L, n, H, D) float32 cached rows at their
    source positions; ``target_idx``: (n,) prompt rows; ``delta``: (n,) int64
    ``target_idx - source_positions`` (pic.py:60-61).
    """

    agent: int
    master_k: np.ndarray
    master_v: np.ndarray
    target_idx: np.ndarray
    delta: np.ndarray


def _rotate_jobs_layer(jobs: Sequence[CollectJob], layer: int, base: float,
                       any_delta: bool) -> np.ndarray:
    stacked = np.concatenate([j.master_k[layer] for j in jobs])
    if not any_delta:
        return stacked
    deltas = np.concatenate([j.delta for j in jobs])
    return rope_apply(stacked, deltas, base)


def collect_into_contexts(jobs: Sequence[CollectJob],
                          contexts: Sequence[Tuple[np.ndarray, np.ndarray]],
                          base: float) -> int:
    """Batched align (pic.py:208-235) plus the skeleton V copy
    (pic.py:203-204): writes rotated K and copied V rows into each agent's
    dense (L, T, H, D) context.  Returns the number of rotation calls (one
    per layer, the ledger law of pic.py:229-230)."""
    if not jobs:
        return 0
    any_delta = any(bool(np.any(j.delta)) for j in jobs)
    layers = jobs[0].master_k.shape[0]
    for j in jobs:
        contexts[j.agent][1][:, j.target_idx] = j.master_v
    for layer in range(layers):
        rotated = _rotate_jobs_layer(jobs, layer, base, any_delta)
        row = 0
        for j in jobs:
            n = j.target_idx.size
            contexts[j.agent][0][layer][j.target_idx] = rotated[row:row + n]
            row += n
    return layers


def collect_into_pool(jobs: Sequence[CollectJob], slot_maps: Sequence[np.ndarray],
                      pool_k: np.ndarray, pool_v: np.ndarray, base: float) -> int:
    """The collector with the pool as its destination: the rows the
    reference first rotates into a dense context (pic.py:234) and later
    copies with PagedPool.write_rows (trace.py:148-152, paged_pool.py:150-156)
    land at ``pool[l, slot_map[agent][target_idx]]``."""
    if not jobs:
        return 0
    any_delta = any(bool(np.any(j.delta)) for j in jobs)
    layers = jobs[0].master_k.shape[0]
    for layer in range(layers):
        rotated = _rotate_jobs_layer(jobs, layer, base, any_delta)
        row = 0
        for j in jobs:
            n = j.target_idx.size
            slots = slot_maps[j.agent][j.target_idx]
            pool_k[layer, slots] = rotated[row:row + n]
            pool_v[layer, slots] = j.master_v[layer]
            row += n
    return layers


# ---------------------------------------------------------------------------
# block-sparse diff codec -- diffstore.py:110-306


class HintViolation(RuntimeError):
    """Mirror differs from master outside the hinted blocks (diffstore.py:156-164)."""


@dataclass
class DiffLayer:
    indices: np.ndarray          # int64, strictly ascending
    k_blocks: np.ndarray         # (count, bs, H, D) float32, zero padded
    v_blocks: np.ndarray
    v_indices: Optional[np.ndarray] = None   # escape form (separate V list)


def _padded(rows: np.ndarray, bs: int) -> np.ndarray:
    out = np.zeros((bs,) + rows.shape[1:], dtype=np.float32)
    out[: rows.shape[0]] = rows
    return out


def encode_diff(master_k: np.ndarray, master_v: np.ndarray,
                mirror_k: np.ndarray, mirror_v: np.ndarray,
                hints: np.ndarray, block_size: int) -> List[DiffLayer]:
    """Restates encode_diff (diffstore.py:119-182): every (layer, block) is
    compared with float equality; changed blocks must be hinted (the first
    violation in layer-major, block-ascending order raises with the block's
    max-abs difference); changed blocks are stored whole, zero-padded."""
    if master_k.shape != mirror_k.shape:
        raise ValueError("master and mirror must have identical plane shapes")
    layers, total, heads, dim = master_k.shape
    nb = block_count(total, block_size)
    hints = np.asarray(hints, dtype=np.int64)
    if hints.size and (hints.min() < 0 or hints.max() >= total):
        raise ValueError("hint positions out of range")
    hinted = np.zeros(nb, dtype=bool)
    hinted[hints // block_size] = True
    out: List[DiffLayer] = []
    for layer in range(layers):
        changed: List[int] = []
        for b in range(nb):
            lo, hi = block_range(b, total, block_size)
            a_k, b_k = mirror_k[layer, lo:hi], master_k[layer, lo:hi]
            a_v, b_v = mirror_v[layer, lo:hi], master_v[layer, lo:hi]
            if np.array_equal(a_k, b_k) and np.array_equal(a_v, b_v):
                continue
            if not hinted[b]:
                worst = max(float(np.abs(a_k - b_k).max()), float(np.abs(a_v - b_v).max()))
                raise HintViolation(
                    f"layer {layer} block {b} differs outside the hinted"
                    f" positions (max abs {worst:.3e})")
            changed.append(b)
        if changed:
            kb = np.stack([_padded(mirror_k[layer, lo:hi], block_size)
                           for lo, hi in (block_range(b, total, block_size) for b in changed)])
            vb = np.stack([_padded(mirror_v[layer, lo:hi], block_size)
                           for lo, hi in (block_range(b, total, block_size) for b in changed)])
        else:
            kb = np.zeros((0, block_size, heads, dim), np.float32)
            vb = np.zeros((0, block_size, heads, dim), np.float32)
        out.append(DiffLayer(np.asarray(changed, dtype=np.int64), kb, vb))
    return out


def _overlay(plane: np.ndarray, idx: np.ndarray, blocks: np.ndarray, bs: int) -> None:
    total = plane.shape[0]
    for j, b in enumerate(idx.tolist()):
        lo, hi = block_range(int(b), total, bs)
        plane[lo:hi] = blocks[j, : hi - lo]


def decode_dense(master_k: np.ndarray, master_v: np.ndarray,
                 layers: Sequence[DiffLayer], block_size: int) -> Tuple[np.ndarray, np.ndarray]:
    """Master copy with the changed blocks overlaid (diffstore.py:185-203)."""
    k, v = master_k.copy(), master_v.copy()
    for layer, ld in enumerate(layers):
        _overlay(k[layer], ld.indices, ld.k_blocks, block_size)
        vidx = ld.indices if ld.v_indices is None else ld.v_indices
        _overlay(v[layer], vidx, ld.v_blocks, block_size)
    return k, v


# wire format (diffstore.py:10-23, 210-306; README "Diff wire format")

_HDR = struct.Struct("<4sHHIIII")


class WireError(ValueError):
    """Malformed serialized diff (diffstore.py:41-42)."""


def wire_size(counts: Sequence[int], block_size: int, heads: int, dim: int) -> int:
    """Bytes of the flag-1 serialization: 24 B header, per layer 5 B plus
    4 B per index plus K and V payload, 4 B trailer."""
    blk = block_size * heads * dim * 4
    return _HDR.size + sum(5 + 4 * c + 2 * c * blk for c in counts) + 4


def serialize(layers: Sequence[DiffLayer], block_size: int, heads: int,
              dim: int, total: int) -> bytes:
    buf = bytearray(_HDR.pack(b"TDDF", 1, len(layers), block_size, heads, dim, total))
    for ld in layers:
        shared = ld.v_indices is None
        buf += struct.pack("<IB", ld.indices.size, 1 if shared else 0)
        buf += ld.indices.astype("<u4").tobytes()
        buf += np.ascontiguousarray(ld.k_blocks, dtype="<f4").tobytes()
        if not shared:
            buf += struct.pack("<I", ld.v_indices.size)
            buf += ld.v_indices.astype("<u4").tobytes()
        buf += np.ascontiguousarray(ld.v_blocks, dtype="<f4").tobytes()
    buf += struct.pack("<I", valid_len(total, block_size))
    return bytes(buf)


def deserialize(buf: bytes):
    """Strict parser: returns (geometry tuple, layers) or raises WireError."""
    pos = 0

    def take(n: int, what: str) -> bytes:
        nonlocal pos
        if pos + n > len(buf):
            raise WireError(f"truncated diff: expected {what}")
        chunk = buf[pos:pos + n]
        pos += n
        return chunk

    magic, ver, nl, bs, h, d, total = _HDR.unpack(take(_HDR.size, "header"))
    if magic != b"TDDF":
        raise WireError("bad magic")
    if ver != 1:
        raise WireError(f"unsupported version {ver}")
    if min(nl, bs, h, d, total) <= 0:
        raise WireError("non-positive geometry field")

    def ids(count: int, what: str) -> np.ndarray:
        a = np.frombuffer(take(4 * count, what), dtype="<u4").astype(np.int64)
        if a.size > 1 and not (np.diff(a) > 0).all():
            raise WireError(f"{what} must be strictly increasing")
        return a

    def blocks(count: int, what: str) -> np.ndarray:
        raw = take(count * bs * h * d * 4, what)
        return np.frombuffer(raw, dtype="<f4").astype(np.float32).reshape(count, bs, h, d)

    layers = []
    for layer in range(nl):
        (count,) = struct.unpack("<I", take(4, f"layer {layer} count"))
        flag = take(1, f"layer {layer} index flag")[0]
        if flag not in (0, 1):
            raise WireError(f"layer {layer}: unknown index flag {flag}")
        idx = ids(count, f"layer {layer} indices")
        kb = blocks(count, f"layer {layer} K payload")
        if flag == 1:
            layers.append(DiffLayer(idx, kb, blocks(count, f"layer {layer} V payload")))
        else:
            (vc,) = struct.unpack("<I", take(4, f"layer {layer} V count"))
            vidx = ids(vc, f"layer {layer} V indices")
            layers.append(DiffLayer(idx, kb, blocks(vc, f"layer {layer} V payload"), vidx))
    (vl,) = struct.unpack("<I", take(4, "valid_len trailer"))
    if pos != len(buf):
        raise WireError("trailing bytes after diff")
    nbk = block_count(total, bs)
    for ld in layers:
        for a in (ld.indices, ld.v_indices):
            if a is not None and a.size and (a.min() < 0 or a.max() >= nbk):
                raise ValueError("block index out of range")
    if vl != valid_len(total, bs):
        raise WireError("valid_len disagrees with token count")
    return (nl, bs, h, d, total), layers


# ---------------------------------------------------------------------------
# restores -- restore.py:29-139


def fused_restore(master_k: np.ndarray, master_v: np.ndarray,
                  layers: Sequence[DiffLayer], block_size: int,
                  old_positions: np.ndarray, new_positions: np.ndarray,
                  slots: np.ndarray, pool_k: np.ndarray, pool_v: np.ndarray,
                  base: float) -> None:
    """Per layer: master planes, diff overlaid BEFORE rotation (restore.py:5-8,
    88), rope_recover on K, rows written to ``pool[l, slots]``."""
    for layer, ld in enumerate(layers):
        k = master_k[layer].copy()
        v = master_v[layer].copy()
        _overlay(k, ld.indices, ld.k_blocks, block_size)
        _overlay(v, ld.indices if ld.v_indices is None else ld.v_indices,
                 ld.v_blocks, block_size)
        pool_k[layer, slots] = rope_recover(old_positions, new_positions, k, base)
        pool_v[layer, slots] = v


def dense_restore(master_k, master_v, layers, block_size, old_positions,
                  new_positions, slots, pool_k, pool_v, base) -> None:
    """Materialize first, then rotate and write (restore.py:107-139)."""
    k, v = decode_dense(master_k, master_v, layers, block_size)
    for layer in range(k.shape[0]):
        pool_k[layer, slots] = rope_recover(old_positions, new_positions, k[layer], base)
        pool_v[layer, slots] = v[layer]


# ---------------------------------------------------------------------------
# family election inputs -- collective.py:117-149


def select_master(scores: dict) -> int:
    """argmin over (score, id) (collective.py:117-121)."""
    if not scores:
        raise ValueError("cannot elect a master from an empty group")
    return sorted(scores.items(), key=lambda kv: (kv[1], kv[0]))[0][0]


def mirror_hints(member_entry: np.ndarray, member_offset: np.ndarray,
                 master_entry: np.ndarray, master_offset: np.ndarray,
                 member_important: np.ndarray, master_important: np.ndarray) -> np.ndarray:
    """Positions where a mirror may differ from its master
    (collective.py:124-149)."""
    if member_entry.size != master_entry.size:
        raise ValueError("hints are only defined for equal-length prompts")
    fresh = (member_entry < 0) | (master_entry < 0)
    moved = (member_entry != master_entry) | (member_offset != master_offset)
    pos = np.flatnonzero(fresh | moved)
    pos = np.union1d(pos, member_important)
    return np.union1d(pos, master_important).astype(np.int64)


# ---------------------------------------------------------------------------
# toy transformer (the selective recompute's arithmetic) -- toymodel.py:26-167


@dataclass
class ToyWeights:
    num_heads: int
    head_dim: int
    rope_base: float
    embed: np.ndarray     # (vocab, hidden)
    wq: np.ndarray        # (layers, hidden, hidden)
    wk: np.ndarray
    wv: np.ndarray
    wm: np.ndarray


def build_weights(num_layers: int, num_heads: int, head_dim: int, vocab_size: int,
                  weight_seed: int = 0, rope_base: float = 10000.0) -> ToyWeights:
    """U[-0.1, 0.1] float32 draws from PCG64(SeedSequence(seed)) in the order
    embedding, then per layer q, k, v, mix (toymodel.py:36-57)."""
    rng = np.random.default_rng(np.random.SeedSequence(weight_seed))
    hid = num_heads * head_dim

    def u(*shape):
        return rng.uniform(-0.1, 0.1, size=shape).astype(np.float32)

    embed = u(vocab_size, hid)
    mats = {name: np.empty((num_layers, hid, hid), np.float32) for name in "qkvm"}
    for layer in range(num_layers):
        for name in "qkvm":
            mats[name][layer] = u(hid, hid)
    return ToyWeights(num_heads, head_dim, rope_base, embed, mats["q"], mats["k"], mats["v"],
                      mats["m"])


def selective_forward(w: ToyWeights, tokens: np.ndarray, positions: np.ndarray,
                      fix_idx: np.ndarray, ctx_k: np.ndarray, ctx_v: np.ndarray,
                      max_layer: Optional[int] = None):
    """Fresh K/V at the ``fix_idx`` rows; other rows come from the context,
    causal by sequence index (toymodel.py:99-151)."""
    layers = w.wq.shape[0] if max_layer is None else max_layer
    H, D = w.num_heads, w.head_dim
    T, F = tokens.shape[0], fix_idx.shape[0]
    out_k = np.empty((layers, F, H, D), np.float32)
    out_v = np.empty_like(out_k)
    if F == 0:
        return out_k, out_v
    pos = positions[fix_idx]
    scale = np.float32(1.0 / np.sqrt(D))
    visible = np.arange(T)[None, :] <= fix_idx[:, None]
    h = w.embed[tokens[fix_idx]]
    for layer in range(layers):
        q = rope_apply((h @ w.wq[layer]).reshape(F, H, D), pos, w.rope_base)
        k = rope_apply((h @ w.wk[layer]).reshape(F, H, D), pos, w.rope_base)
        v = (h @ w.wv[layer]).reshape(F, H, D)
        out_k[layer], out_v[layer] = k, v
        keys = ctx_k[layer].copy()
        vals = ctx_v[layer].copy()
        keys[fix_idx], vals[fix_idx] = k, v
        s = np.einsum("fhd,thd->hft", q, keys) * scale
        s = np.where(visible[None], s, np.float32(-np.inf))
        p = np.exp(s - s.max(axis=-1, keepdims=True))
        p /= p.sum(axis=-1, keepdims=True)
        h = h + np.einsum("hft,thd->fhd", p, vals).reshape(F, H * D) @ w.wm[layer]
    return out_k, out_v


def full_prefill(w: ToyWeights, tokens, start_pos: int = 0):
    """All rows fresh at positions start_pos.. (toymodel.py:154-167)."""
    toks = np.asarray(tokens, np.int64)
    T = toks.size
    L, H, D = w.wq.shape[0], w.num_heads, w.head_dim
    zeros = np.zeros((L, T, H, D), np.float32)
    pos = np.arange(start_pos, start_pos + T, dtype=np.int64)
    return selective_forward(w, toks, pos, np.arange(T), zeros, zeros)


def key_diff(fresh: np.ndarray, cached: np.ndarray) -> np.ndarray:
    """Per-position L2 norm of the float32 key difference (pic.py:166-171)."""
    if fresh.shape != cached.shape:
        raise ValueError("key tensors must have identical shapes")
    diff = (fresh - cached).reshape(fresh.shape[0], -1)
    return np.sqrt(np.einsum("te,te->t", diff, diff))


def select_important(mags: np.ndarray, budget: int) -> np.ndarray:
    """Largest magnitudes first, ties to the lower index, zeros excluded,
    result sorted ascending (pic.py:180-189)."""
    if mags.size == 0 or budget <= 0:
        return np.empty(0, dtype=np.int64)
    idx = np.arange(mags.size)
    ranked = idx[np.lexsort((idx, -mags))]
    ranked = ranked[mags[ranked] > 0.0][:budget]
    return np.sort(ranked).astype(np.int64)


def recompute_budget(fraction: float, shared_count: int) -> int:
    """ceil(fraction*shared) with decimal-noise guard (pic.py:174-177)."""
    return int(math.ceil(round(fraction * shared_count, 6)))


# ---------------------------------------------------------------------------
# segment index (segment_index.py:86-183)


class SegmentIndexPort:
    """Digest -> entries cache with byte-budget LRU eviction, restated from
    segment_index.SegmentIndex: per digest a stack of entries (lookup takes
    the newest, :125-135); recency = insertion-ordered map keyed by entry_id,
    refreshed by lookup (:131-134); insert adds then evicts to the budget
    (:137-143); eviction walks oldest-first, skipping pinned refs, until the
    total fits (:159-170); removal subtracts the size and reports on_evict
    even for an entry that is not present (:172-181)."""

    def __init__(self, budget_bytes, is_pinned=None, on_evict=None):
        if budget_bytes < 0:
            raise ValueError("budget must be non-negative")
        self.budget_bytes = int(budget_bytes)
        self.is_pinned = is_pinned or (lambda ref: False)
        self.on_evict = on_evict
        self.stacks = {}
        self.order = {}
        self.total = 0

    def __len__(self):
        return len(self.order)

    def __contains__(self, digest):
        return bool(self.stacks.get(digest))

    @property
    def total_bytes(self):
        return self.total

    def entries(self):
        return tuple(self.order.values())

    def lookup(self, digest):
        stack = self.stacks.get(digest)
        if not stack:
            return None
        e = stack[-1]
        self.order.pop(e.entry_id, None)
        self.order[e.entry_id] = e
        return e

    def insert(self, e):
        self.stacks.setdefault(e.digest, []).append(e)
        self.order[e.entry_id] = e
        self.total += e.nbytes
        self._evict(self.budget_bytes)

    def remove(self, e):
        if self.is_pinned(e.kv_ref):
            raise RuntimeError("entry is pinned by live mirrors")
        self._drop(e)

    def evict_to_budget(self, budget=None):
        return self._evict(self.budget_bytes if budget is None else budget)

    def _evict(self, budget):
        n = 0
        for e in list(self.order.values()):
            if self.total <= budget:
                break
            if self.is_pinned(e.kv_ref):
                continue
            self._drop(e)
            n += 1
        return n

    def _drop(self, e):
        stack = self.stacks.get(e.digest, [])
        if e in stack:
            stack.remove(e)
            if not stack:
                del self.stacks[e.digest]
        self.order.pop(e.entry_id, None)
        self.total -= e.nbytes
        if self.on_evict is not None:
            self.on_evict(e)


# ---------------------------------------------------------------------------
# request preparation (pic.py:110-163, core.py:120-140)


@dataclass
class PreparedPort:
    tokens: np.ndarray
    private_idx: np.ndarray
    structural_idx: np.ndarray
    hits: list                   # [(entry, target_idx)]
    label_entry: np.ndarray
    label_offset: np.ndarray


def prepare_request_port(segments, separator: int, lookup) -> PreparedPort:
    """Restates prepare_request (pic.py:110-163) over a list of
    (kind, tokens, digest) segments: flatten with one separator between
    consecutive segments (core.py:130-140; a separator inside a segment is a
    ValueError), the private history is the first segment's range, every
    SHARED segment is looked up (``lookup(digest)`` -> entry or None, in
    segment order), a hit labels its positions with (entry.entry_id, offset),
    a miss or a task segment is structural, and so is the separator before
    every segment after the first."""
    for _, toks, _ in segments:
        if separator in toks:
            raise ValueError("separator id must not occur inside a segment")
    flat = []
    starts = []
    for i, (_, toks, _) in enumerate(segments):
        if i:
            flat.append(int(separator))
        starts.append(len(flat))
        flat.extend(int(t) for t in toks)
    total = len(flat)
    label_entry = np.full(total, -1, np.int64)
    label_offset = np.full(total, -1, np.int64)
    private = np.empty(0, np.int64)
    structural, hits = [], []
    for (kind, toks, digest), start in zip(segments, starts):
        idx = np.arange(start, start + len(toks), dtype=np.int64)
        if kind == "private_history":
            private = idx
            continue
        entry = lookup(digest) if kind == "shared_output" else None
        if entry is None:
            structural.extend(idx.tolist())
            continue
        hits.append((entry, idx))
        label_entry[idx] = entry.entry_id
        label_offset[idx] = np.arange(len(toks))
    structural.extend(s - 1 for s in starts[1:])
    return PreparedPort(np.asarray(flat, np.int64), private,
                        np.asarray(sorted(structural), np.int64), hits, label_entry,
                        label_offset)
