"""Selective recompute of deviating tokens on the B200 (reference:
roundkv/toymodel.py:99-192 and pic.refresh, pic.py:284-300).

The reference recomputes the important and structural rows of a prompt
with its seeded toy transformer (embedding, per layer Q/K/V projections
with rotary Q/K, causal softmax attention over the partly cached context,
output mix folded into the residual stream; float32).  Here every
projection is a tensor-core GEMM (``tdkv_gemm``: tcgen05, TMEM accumulator,
3xTF32 for float32 operands), the rotary step and the attention are
``tdkv_qkv_rope`` / ``tdkv_attention_many`` (query-tiled; online softmax for
head_dim <= 128), and the embedding gather and the row write-back use the row
mover (K3).  The final layer's attention and mix are skipped: their only
consumer is the next layer.  ``forward_many`` runs several requests' forwards
as one batch (grouped recovery); ``selective_forward`` is its one-request
case.

Signatures follow the reference: ``selective_forward`` (= _selective_forward),
``full_prefill``, ``recompute_positions`` and ``refresh``; ``weights`` is the
reference's ``ModelWeights`` (or anything with ``config``, ``embed``,
``wq/wk/wv/wm``).
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _kernels, _lib
from ._device import default_device, h2d, is_host, ptr, stream_handle, to_device, to_host
from .core import LayeredKv, ModelConfig, union_sorted
from .gemm import gemm_tf32x3, gemm_tn, tf32_split
from .ledger import CostLedger


@dataclass(eq=False)
class ModelWeights:
    """The toy transformer's weights (toymodel.py:26-33): embedding (vocab,
    hidden) and per-layer q / k / v / mix matrices (layers, hidden, hidden),
    float32 on the host; ``ToyModel.of`` keeps the device copies."""

    config: ModelConfig
    embed: np.ndarray
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wm: np.ndarray


def build_weights(config: ModelConfig) -> ModelWeights:
    """U[-0.1, 0.1] float32 draws from one PCG64(SeedSequence(weight_seed))
    stream in the reference's order -- embedding, then per layer q, k, v, mix
    (toymodel.py:36-57) -- so the weights are the reference's bit for bit."""
    rng = np.random.default_rng(np.random.SeedSequence(config.weight_seed))
    hid = config.hidden_dim

    def draw(*shape: int) -> np.ndarray:
        return rng.uniform(-0.1, 0.1, size=shape).astype(np.float32)

    embed = draw(config.vocab_size, hid)
    mats = [np.empty((config.num_layers, hid, hid), dtype=np.float32) for _ in range(4)]
    for layer in range(config.num_layers):
        for mat in mats:
            mat[layer] = draw(hid, hid)
    return ModelWeights(config, embed, *mats)


def _cfg(weights):
    cfg = getattr(weights, "config", weights)
    return (int(cfg.num_layers if hasattr(cfg, "num_layers") else weights.wq.shape[0]),
            int(cfg.num_heads), int(cfg.head_dim), float(getattr(cfg, "rope_base", 10000.0)))


class ToyModel:
    """Device-resident weights: embedding, [Wq|Wk|Wv]^T per layer (3*hid, hid)
    and Wm^T per layer (hid, hid), all float32 (K-major GEMM operands)."""

    _cache: dict = {}

    def __init__(self, weights, device: torch.device) -> None:
        self.num_layers, self.num_heads, self.head_dim, self.rope_base = _cfg(weights)
        hid = self.num_heads * self.head_dim
        if hid % 4:
            raise ValueError("hidden size must be a multiple of 4 (16-byte GEMM rows)")
        self.hidden = hid
        self.device = device
        self.embed = to_device(np.asarray(weights.embed, np.float32), device)
        wq, wk, wv, wm = (np.asarray(getattr(weights, n), np.float32) for n in ("wq", "wk", "wv", "wm"))
        qkv_t = np.concatenate([wq.transpose(0, 2, 1), wk.transpose(0, 2, 1),
                                wv.transpose(0, 2, 1)], axis=1)
        self.wqkv_t = to_device(np.ascontiguousarray(qkv_t), device)
        self.wm_t = to_device(np.ascontiguousarray(wm.transpose(0, 2, 1)), device)
        # the weights' tf32 hi / lo planes, split once (3xTF32 GEMMs over
        # pre-split operands); TDKV_GEMM_PRESPLIT=0 splits inside every GEMM
        self.presplit = _PRESPLIT
        if self.presplit:
            self.wqkv_t_split = tf32_split(self.wqkv_t)
            self.wm_t_split = tf32_split(self.wm_t)

    @classmethod
    def of(cls, weights, device: Optional[torch.device] = None) -> "ToyModel":
        if isinstance(weights, ToyModel):
            return weights
        device = device or default_device()
        key = (id(weights), device)
        m = cls._cache.get(key)
        if m is None or m._src is not weights:
            m = cls(weights, device)
            m._src = weights
            cls._cache[key] = m
        return m


def selective_forward(weights, tokens, positions, fix_idx, ctx_k, ctx_v,
                      max_layer: Optional[int] = None):
    """Fresh K/V rows at ``fix_idx`` against the cached context; returns
    (k, v) of shape (layers_run, F, H, D) -- numpy for numpy contexts."""
    host = is_host(ctx_k)
    dev = ctx_k.device if isinstance(ctx_k, torch.Tensor) else default_device()
    m = ToyModel.of(weights, dev)
    H, D, hid = m.num_heads, m.head_dim, m.hidden
    toks = np.asarray(tokens, np.int64)
    pos = np.asarray(positions, np.int64)
    fix = np.asarray(fix_idx, np.int64)
    T, F = toks.size, fix.size
    layers = m.num_layers if max_layer is None else int(max_layer)
    if F and layers:
        ck = to_device(ctx_k, dev, torch.float32)
        cv = to_device(ctx_v, dev, torch.float32)
        out_k, out_v, _ = forward_many(m, [(toks, pos, fix, ck, cv)], layers)
    else:
        out_k = torch.empty((layers, F, H, D), dtype=torch.float32, device=dev)
        out_v = torch.empty_like(out_k)
    if host:
        return to_host(out_k), to_host(out_v)
    return out_k, out_v


_PRESPLIT = os.environ.get("TDKV_GEMM_PRESPLIT", "1") != "0"

# TDKV_ATTN_ONLINE=0 keeps the two-pass (stored score row) attention everywhere
_ATTN_ONLINE = os.environ.get("TDKV_ATTN_ONLINE", "1") != "0"


# TDKV_ATTN_BLOCK=0 keeps the 16-row online kernel for head dims the
# register-blocked 64-row kernel serves
_ATTN_BLOCK = os.environ.get("TDKV_ATTN_BLOCK", "1") != "0"


# TDKV_ATTN_TC=0 keeps the CUDA-core kernels for head dims the tensor-core
# attention serves
_ATTN_TC = os.environ.get("TDKV_ATTN_TC", "1") != "0"


def _attn_rows_per_tile(head_dim: int) -> int:
    """Fixed rows per CTA of the query-tiled attention: 128 with the
    tensor-core kernel (head_dim 32 or 64: tcgen05 3xTF32 for Q K^T and P V),
    64 with the register-blocked kernel (head_dim 8, 16, 32, 64 or 128), else
    16 with the online softmax (head_dim <= 128), else 8."""
    if _ATTN_TC and _ATTN_ONLINE and head_dim in (32, 64):
        return 128
    if _ATTN_BLOCK and _ATTN_ONLINE and head_dim in (8, 16, 32, 64, 128):
        return 64
    return 16 if _ATTN_ONLINE and head_dim <= 128 else 8


def forward_many(m: ToyModel, items, layers: int, k_only_last: bool = False):
    """The selective forward of several independent requests as ONE batch:
    ``items`` = [(tokens, positions, fix_idx, ctx_k, ctx_v)] (host integer
    arrays; device float32 context planes of shape (L, T_i, H, D), or None
    when every attended row is fresh).  Per layer one QKV GEMM, one rotary
    launch, one attention launch and one mix GEMM cover every item's fixed
    rows (grouped recovery, collective.py:152-187, batches its members this
    way); row results do not depend on the batch (rows are independent in
    the GEMMs and attend only to their own item's context).

    ``k_only_last``: the caller reads only K of the last layer (the probe's
    check layer), so that layer projects K alone (a third of its QKV GEMM);
    its V plane is then undefined.

    Returns (out_k, out_v, row0): planes (layers, sum F_i, H, D) with item i's
    rows at [row0[i], row0[i] + F_i)."""
    dev = m.device
    H, D, hid = m.num_heads, m.head_dim, m.hidden
    fixes = [np.asarray(it[2], np.int64) for it in items]
    F = np.array([f.size for f in fixes], np.int64)
    row0 = np.concatenate([[0], np.cumsum(F)[:-1]]).astype(np.int64)
    R = int(F.sum())
    out_k = torch.empty((layers, max(R, 1), H, D), dtype=torch.float32, device=dev)
    out_v = torch.empty_like(out_k)
    if R == 0 or layers == 0:
        return out_k, out_v, row0
    toks = [np.asarray(it[0], np.int64) for it in items]
    pos = [np.asarray(it[1], np.int64) for it in items]
    Ts = [t.size for t in toks]
    # ONE upload per forward: [fix indices | tokens | positions (int64, R each) |
    # attention member table | fresh_of maps (int32)]; device addresses inside
    # the table point back into the same buffer
    sumT = int(sum(Ts))
    live = F > 0
    n_live = int(live.sum())
    mt = _lib.ATTN_MEMBER.itemsize
    nbytes = 24 * R + mt * n_live + 4 * sumT
    d_blob = torch.empty(nbytes + 8, dtype=torch.uint8, device=dev)
    base = ptr(d_blob)
    fix_base, tok_base, pos_base = base, base + 8 * R, base + 16 * R
    mem_base = base + 24 * R
    fo_base = mem_base + mt * n_live
    blob = np.zeros(nbytes, np.uint8)
    i64 = blob[:24 * R].view(np.int64)
    i64[:R] = np.concatenate(fixes)
    i64[R:2 * R] = np.concatenate([t[f] for t, f in zip(toks, fixes)])
    i64[2 * R:] = np.concatenate([p[f] for p, f in zip(pos, fixes)])
    fresh_of = blob[24 * R + mt * n_live:].view(np.int32)
    fresh_of[:] = -1
    t0 = np.concatenate([[0], np.cumsum(Ts)[:-1]]).astype(np.int64)
    for i, f in enumerate(fixes):
        fresh_of[t0[i] + f] = np.arange(f.size, dtype=np.int32)
    rows_per_tile = _attn_rows_per_tile(D)
    tiles = -(-F // rows_per_tile)                # query tiles per member
    tile0 = np.concatenate([[0], np.cumsum(tiles)[:-1]]).astype(np.int64)
    n_tiles = int(tiles.sum()) if D <= 128 else 0
    members = blob[24 * R:24 * R + mt * n_live].view(_lib.ATTN_MEMBER)
    j = 0
    for i, it in enumerate(items):
        if not live[i]:
            continue
        ck, cv = it[3], it[4]
        if ck is None:                       # every attended row is fresh: never read
            ck = cv = out_k
            stride = 0
        else:
            stride = int(ck.shape[1]) * hid
        members[j] = (ptr(ck), ptr(cv), fo_base + 4 * int(t0[i]), fix_base + 8 * int(row0[i]),
                      stride, int(row0[i]), int(F[i]), Ts[i], int(tile0[i]))
        j += 1
    staged = torch.from_numpy(blob).pin_memory()
    d_blob[:nbytes].copy_(staged, non_blocking=True)
    d_i64 = d_blob[:24 * R].view(torch.int64)
    table = torch.empty((R, D // 2, 2), dtype=torch.float64, device=dev)
    _kernels.rope_table_from_device(d_i64[2 * R:], D, m.rope_base, torch.float32, table)
    h = torch.empty((R, hid), dtype=torch.float32, device=dev)
    job = _kernels.rows_job(m.embed, None, 0, h, None, 0, R, src_rows=d_i64[R:2 * R])
    _kernels.rows(_kernels.rows_jobs([job]), R, None, 1, 1, hid, _kernels.ROWS_BLOCK,
                  torch.float32, dev)
    qkv = torch.empty((R, 3 * hid), dtype=torch.float32, device=dev)
    q = torch.empty((R, hid), dtype=torch.float32, device=dev)
    mix = torch.empty((R, hid), dtype=torch.float32, device=dev)
    d_members = mem_base
    scale = float(np.float32(1.0 / np.sqrt(D)))
    stream = stream_handle(dev)
    if m.presplit:
        a_split = (torch.empty((R, hid), dtype=torch.float32, device=dev),
                   torch.empty((R, hid), dtype=torch.float32, device=dev))
    for layer in range(layers):
        if m.presplit:
            tf32_split(h, out=a_split)
            wh, wl = m.wqkv_t_split[0][layer], m.wqkv_t_split[1][layer]
            if k_only_last and layer == layers - 1:
                gemm_tf32x3(a_split, (wh[hid:2 * hid], wl[hid:2 * hid]), out=qkv[:, hid:2 * hid])
            else:
                gemm_tf32x3(a_split, (wh, wl), out=qkv)
        elif k_only_last and layer == layers - 1:
            # K columns only; Q and V of this layer are never read
            gemm_tn(h, m.wqkv_t[layer][hid:2 * hid], out=qkv[:, hid:2 * hid])
        else:
            gemm_tn(h, m.wqkv_t[layer], out=qkv)
        _lib.call("tdkv_qkv_rope", ptr(qkv), ptr(table), R, H, D, ptr(q), ptr(out_k[layer]),
                  ptr(out_v[layer]), stream)
        if layer == layers - 1:
            break                       # the last layer's attention only feeds h
        _lib.call("tdkv_attention_many", ptr(q), ptr(out_k[layer]), ptr(out_v[layer]),
                  d_members, n_live, layer, R, n_tiles, rows_per_tile, max(Ts), H, D,
                  scale, ptr(mix), stream)
        if m.presplit:
            tf32_split(mix, out=a_split)
            gemm_tf32x3(a_split, (m.wm_t_split[0][layer], m.wm_t_split[1][layer]), out=h,
                        accumulate=True)
        else:
            gemm_tn(mix, m.wm_t[layer], out=h, accumulate=True)
    return out_k, out_v, row0


def full_prefill(weights, tokens: Sequence[int], start_pos: int = 0) -> LayeredKv:
    """Ground-truth prefill of every row (toymodel.py:154-167), on the device;
    returns host float32 planes like the reference."""
    toks = np.asarray(tokens, dtype=np.int64)
    L, H, D, _ = _cfg(weights)
    vocab = int(np.asarray(weights.embed).shape[0])
    if toks.ndim != 1 or toks.size == 0:
        raise ValueError("tokens must be one non-empty sequence")
    if toks.min() < 0 or toks.max() >= vocab:
        raise ValueError("token id out of vocabulary range")
    T = toks.size
    positions = np.arange(start_pos, start_pos + T, dtype=np.int64)
    zeros = np.zeros((L, T, H, D), np.float32)
    k, v = selective_forward(weights, toks, positions, np.arange(T), zeros, zeros)
    return LayeredKv(k, v, positions)


def recompute_positions(weights, tokens, positions_to_fix, context_kv: LayeredKv):
    """(sorted fix indices, k rows, v rows) against a cached context
    (toymodel.py:170-192)."""
    toks = np.asarray(tokens, dtype=np.int64)
    if toks.shape[0] != context_kv.num_tokens:
        raise ValueError("context must cover the full token sequence")
    L = _cfg(weights)[0]
    if context_kv.num_layers != L:
        raise ValueError("context layer count does not match the model")
    fix = np.unique(np.asarray(list(positions_to_fix), dtype=np.int64))
    if fix.size and (fix[0] < 0 or fix[-1] >= toks.shape[0]):
        raise ValueError("fix index out of range")
    k, v = selective_forward(weights, toks, context_kv.positions, fix, context_kv.k,
                             context_kv.v)
    return fix, k, v


def refresh(weights, prep, context, important: np.ndarray,
            ledger: Optional[CostLedger] = None) -> None:
    """Recompute important and structural positions together at all layers
    and write them into the member's context (pic.py:284-300)."""
    fix = union_sorted(important, prep.structural_idx)
    if fix.size == 0:
        return
    ctx_k, ctx_v = context
    k, v = selective_forward(weights, prep.tokens, prep.positions, fix, ctx_k, ctx_v)
    if is_host(ctx_k):
        ctx_k[:, fix] = k
        ctx_v[:, fix] = v
    else:
        L, F, H, D = k.shape
        T = int(ctx_k.shape[1])
        d_fix = h2d(fix, ctx_k.device)
        job = _kernels.rows_job(k, v, F * H * D, ctx_k, ctx_v, T * H * D, F, dst_rows=d_fix)
        _kernels.rows(_kernels.rows_jobs([job]), F, None, L, H, D, _kernels.ROWS_BLOCK,
                      ctx_k.dtype, ctx_k.device)
    if ledger is not None:
        ledger.record_recomputed(int(fix.size))
