"""Diff-aware storage: block-sparse diffs, wire format, families
(reference: roundkv/diffstore.py).

Encoding (``encode_diff`` / ``encode_batch`` / ``DiffStore.encode_family``)
runs kernel K2 on the device: one compare pass over every (mirror, layer,
block) with float '!=' semantics (diffstore.py:151-153) and one compaction
that writes each layer's changed blocks in ascending order, zero-padded, into
a payload slab (diffstore.py:166-173).  A whole family is encoded in one
launch and one device->host read of the counts and indices.

Decoding is fused into restores (restore.py); ``diff_decode_dense`` is the
dense baseline (diffstore.py:185-203), one K3 launch.

The wire format (diffstore.py:10-23, 210-306) is byte-identical to the
reference's (version 1, float32 payload): encoder output is packed on the GPU
(tdkv_wire_pack, one D2H per batch of diffs) and an image can be unpacked
straight into device slabs for the fused restore (tdkv_wire_unpack); host
diffs keep the host path.
"""
from __future__ import annotations

import struct
import threading
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _kernels, _lib
from ._device import (bytes_to_device, default_device, release_inflight, dtype_code, h2d, ptr, stream_handle,
                      to_device, to_host, upload)
from .core import CacheBlockConfig, LayeredKv, kv_dense_nbytes

MAGIC = b"TDDF"
VERSION = 1
# single-pass encoder (tdkv_diff_encode); TDKV_TWO_PASS_ENCODE=1 selects the
# compare + compact pair
_SINGLE_PASS = not __import__("os").environ.get("TDKV_TWO_PASS_ENCODE")
_HEADER = struct.Struct("<4sHHIIII")


class MalformedDiffError(ValueError):
    """A serialized diff is truncated or inconsistent."""


class HintSoundnessError(RuntimeError):
    """Master and mirror differ outside the hinted positions."""


class PinnedMasterError(RuntimeError):
    """A family whose master has live mirrors was dropped."""


def _nbytes(x) -> int:
    if isinstance(x, torch.Tensor):
        return x.numel() * x.element_size()
    return int(x.nbytes)


def _payload_ok(x, want) -> bool:
    if tuple(x.shape) != want:
        return False
    if isinstance(x, np.ndarray):
        return x.dtype == np.float32
    return isinstance(x, torch.Tensor) and x.dtype in (torch.float32, torch.bfloat16)


@dataclass(eq=False)
class LayerDiff:
    """Changed blocks of one layer; ``v_indices`` None = K and V share
    ``indices`` (the only form the encoder emits)."""

    indices: np.ndarray
    k_blocks: object
    v_blocks: object
    v_indices: Optional[np.ndarray] = None

    def __post_init__(self) -> None:
        self.indices = np.asarray(self.indices, dtype=np.int64)
        if self.v_indices is not None:
            self.v_indices = np.asarray(self.v_indices, dtype=np.int64)

    @property
    def payload_nbytes(self) -> int:
        return _nbytes(self.k_blocks) + _nbytes(self.v_blocks)


@dataclass
class _DeviceDiff:
    """Device form used by the fused decoder: payload slabs + block maps."""

    pay_k: torch.Tensor
    pay_v: torch.Tensor
    map_k: torch.Tensor          # (L * nb) int32, -1 = take the master block
    map_v: torch.Tensor


class _EncodedSlab:
    """Encoder output kept in its device layout: layer l's changed blocks are
    slab rows [l*cap, l*cap + counts[l]) with block ids idx[l*cap:...].  The
    mirror's views of the family tensors are cut on first use (an encode of
    a 49-mirror family then builds no tensor views on the host)."""

    __slots__ = ("counts", "idx", "cap", "_fam", "_row0", "_map", "_map_n", "_views")

    def __init__(self, counts, idx, cap, fam_k, fam_v, row0, fam_map, map0, map_n):
        self.counts = counts         # (L,) int
        self.idx = idx               # (L*cap,) int32, host copy
        self.cap = cap
        self._fam = (fam_k, fam_v, fam_map)
        self._row0 = row0
        self._map = map0
        self._map_n = map_n
        self._views = None

    def _cut(self):
        if self._views is None:
            fk, fv, fm = self._fam
            r0, n = self._row0, self.cap * len(self.counts)
            mp = fm[self._map:self._map + self._map_n]
            self._views = (fk[r0:r0 + n], fv[r0:r0 + n], mp)
        return self._views

    @property
    def pay_k(self) -> torch.Tensor:    # (L*cap, bs, H, D)
        return self._cut()[0]

    @property
    def pay_v(self) -> torch.Tensor:
        return self._cut()[1]

    @property
    def elt_size(self) -> int:
        return self._fam[0].element_size()

    def device_diff(self) -> _DeviceDiff:
        k, v, mp = self._cut()
        return _DeviceDiff(k, v, mp, mp)


class BlockSparseDiff:
    """Per-layer changed blocks of a mirror relative to its master.

    Constructed from ``layers`` (validated like diffstore.py:84-99), or by the
    encoder from its device slab, in which case the per-layer ``LayerDiff``
    views are only materialized when ``layers`` is first read.
    """

    def __init__(self, num_layers: int, block_size: int, num_heads: int, head_dim: int,
                 total_tokens: int, layers: List[LayerDiff]) -> None:
        self.num_layers = num_layers
        self.block_size = block_size
        self.num_heads = num_heads
        self.head_dim = head_dim
        self.total_tokens = total_tokens
        self._layers = list(layers)
        self._slab: Optional[_EncodedSlab] = None
        self._dev: Optional[_DeviceDiff] = None
        if len(self._layers) != self.num_layers:
            raise ValueError("one LayerDiff per layer required")
        nb = CacheBlockConfig(self.block_size).num_blocks(self.total_tokens)
        for ld in self._layers:
            for idx, payload in ((ld.indices, ld.k_blocks), (ld.v_indices, ld.v_blocks)):
                idx = ld.indices if idx is None else idx
                if idx.size and (idx.min() < 0 or idx.max() >= nb):
                    raise ValueError("block index out of range")
                if idx.size > 1 and not (np.diff(idx) > 0).all():
                    raise ValueError("block indices must be strictly increasing")
                want = (idx.size, self.block_size, self.num_heads, self.head_dim)
                if not _payload_ok(payload, want):
                    raise ValueError("payload must be float32 with one block per index")

    @classmethod
    def _from_slab(cls, num_layers: int, block_size: int, num_heads: int, head_dim: int,
                   total_tokens: int, slab: _EncodedSlab,
                   dev: Optional[_DeviceDiff] = None) -> "BlockSparseDiff":
        self = cls.__new__(cls)
        self.num_layers = num_layers
        self.block_size = block_size
        self.num_heads = num_heads
        self.head_dim = head_dim
        self.total_tokens = total_tokens
        self._layers = None
        self._slab = slab
        self._dev = dev
        return self

    @property
    def layers(self) -> List[LayerDiff]:
        if self._layers is None:
            s = self._slab
            out = []
            for layer in range(self.num_layers):
                n = int(s.counts[layer])
                base = layer * s.cap
                out.append(LayerDiff(s.idx[base:base + n].astype(np.int64),
                                     s.pay_k[base:base + n], s.pay_v[base:base + n]))
            self._layers = out
        return self._layers

    @layers.setter
    def layers(self, value: List[LayerDiff]) -> None:
        self._layers = list(value)
        self._slab = None            # the encoder's device form no longer describes it
        self._dev = None

    @property
    def payload_nbytes(self) -> int:
        if self._layers is None:
            s = self._slab
            blk = self.block_size * self.num_heads * self.head_dim * s.elt_size
            return int(2 * blk * int(s.counts.sum()))
        return sum(ld.payload_nbytes for ld in self._layers)

    @property
    def changed_blocks_per_layer(self) -> List[int]:
        if self._layers is None:
            return [int(c) for c in self._slab.counts]
        return [int(ld.indices.size) for ld in self._layers]

    def _plane_counts(self):
        """Per layer (k_count, v_count, escape)."""
        if self._layers is None:
            return [(int(c), int(c), False) for c in self._slab.counts]
        return [(int(ld.indices.size),
                 int(ld.indices.size if ld.v_indices is None else ld.v_indices.size),
                 ld.v_indices is not None) for ld in self._layers]

    def to_host(self) -> "BlockSparseDiff":
        """Bring the payload to host numpy (the reference's representation)."""
        for ld in self.layers:
            if isinstance(ld.k_blocks, torch.Tensor):
                ld.k_blocks = to_host(ld.k_blocks)
            if isinstance(ld.v_blocks, torch.Tensor):
                ld.v_blocks = to_host(ld.v_blocks)
        return self

    def device_form(self, device: torch.device, dtype: torch.dtype) -> _DeviceDiff:
        """Payload slabs + block maps on the device (uploaded once for host diffs)."""
        if self._dev is None and self._slab is not None:
            self._dev = self._slab.device_diff()
        d = self._dev
        if d is not None and d.pay_k.device == device and d.pay_k.dtype == dtype:
            return d
        nb = CacheBlockConfig(self.block_size).num_blocks(self.total_tokens)
        maps = []
        slabs = []
        for plane in ("k", "v"):
            blocks, mp = [], np.full((self.num_layers, nb), -1, np.int32)
            off = 0
            for layer, ld in enumerate(self.layers):
                idx = ld.indices if (plane == "k" or ld.v_indices is None) else ld.v_indices
                payload = ld.k_blocks if plane == "k" else ld.v_blocks
                if idx.size:
                    mp[layer, idx] = np.arange(off, off + idx.size, dtype=np.int32)
                    blocks.append(to_device(payload, device, dtype))
                off += idx.size
            shape = (max(off, 1), self.block_size, self.num_heads, self.head_dim)
            slab = torch.cat(blocks) if blocks else torch.zeros(shape, dtype=dtype, device=device)
            slabs.append(slab)
            maps.append(h2d(mp.reshape(-1), device))
        d = _DeviceDiff(slabs[0], slabs[1], maps[0], maps[1])
        self._dev = d
        return d


# ---------------------------------------------------------------------------
# encoder (K2)


def _check_pair(master: LayeredKv, mirror: LayeredKv) -> None:
    if tuple(master.k.shape) != tuple(mirror.k.shape):
        raise ValueError("master and mirror must have identical plane shapes")
    if not np.array_equal(master.positions, mirror.positions):
        raise ValueError("master and mirror must cover the same positions")


def _plane_dtype(kv: LayeredKv) -> torch.dtype:
    return kv.k.dtype if isinstance(kv.k, torch.Tensor) else torch.float32


def encode_launch(master: LayeredKv, mirrors: Sequence[LayeredKv],
                  hint_positions: Sequence[np.ndarray], blocks: CacheBlockConfig,
                  device: Optional[torch.device] = None) -> "_EncodeState":
    """Validate, upload the descriptors and launch K2 for a family without
    reading anything back; ``encode_finish`` completes it."""
    if len(mirrors) != len(hint_positions) or not mirrors:
        raise ValueError("one hint array per mirror, at least one mirror")
    total = master.num_tokens
    nb = blocks.num_blocks(total)
    bs = blocks.block_size
    L, H, D = master.num_layers, master.num_heads, master.head_dim
    hinted = np.zeros((len(mirrors), nb), np.uint8)
    shape = tuple(master.k.shape)
    if any(tuple(mir.k.shape) != shape for mir in mirrors):
        raise ValueError("master and mirror must have identical plane shapes")
    mpos = np.asarray(master.positions)
    # LayeredKv positions are strictly increasing: two such vectors of one
    # length spanning the same contiguous range [a, a + T) are equal, so the
    # common case needs no element compare; otherwise compare the bytes
    mcontig = mpos.size > 0 and int(mpos[-1]) - int(mpos[0]) == mpos.size - 1
    mbytes = None
    for mir in mirrors:
        pos = mir.positions
        if pos is mpos:
            continue
        pos = np.asarray(pos)
        if (mcontig and pos.shape == mpos.shape and int(pos[0]) == int(mpos[0])
                and int(pos[-1]) == int(mpos[-1])):
            continue
        if mbytes is None:
            mbytes = mpos.tobytes()
        same = (pos.tobytes() == mbytes if pos.dtype == mpos.dtype and pos.shape == mpos.shape
                else np.array_equal(pos, mpos))
        if not same:
            raise ValueError("master and mirror must cover the same positions")
    # every mirror's hint positions -> its hinted-block row: one flat scatter
    # of (mirror * nb + block) over the concatenated hints
    hs = [np.asarray(h).reshape(-1) for h in hint_positions]
    sizes = np.fromiter((h.size for h in hs), np.int64, len(hs))
    if sizes.sum():
        cat = np.concatenate(hs)
        if cat.dtype.kind not in "iu":
            cat = cat.astype(np.int64)
        if cat.min() < 0 or cat.max() >= total:
            raise ValueError("hint positions out of range")
        blk = (cat >> (bs.bit_length() - 1)) if bs & (bs - 1) == 0 else cat // bs
        hinted.reshape(-1)[blk + np.repeat(np.arange(len(hs), dtype=np.int64) * nb, sizes)] = 1
    device = device or (master.k.device if master.on_device else default_device())
    dtype = _plane_dtype(master)
    mk = to_device(master.k, device, dtype)
    mv = to_device(master.v, device, dtype)
    mirrors_dev = [(to_device(m.k, device, dtype), to_device(m.v, device, dtype)) for m in mirrors]
    P = len(mirrors)
    caps = np.maximum(hinted.sum(axis=1).astype(np.int64), 1)
    slab_blocks = int((caps * L).sum())
    # one int32 buffer for everything the host reads back: one D2H copy
    meta = torch.empty(P + P * L + slab_blocks, dtype=torch.int32, device=device)
    violation = meta[:P]
    counts = meta[P:P + P * L]
    indices = meta[P + P * L:]
    changed = None if _SINGLE_PASS else torch.empty(P * L * nb, dtype=torch.uint8, device=device)
    viol_maxabs = torch.empty(P * L * nb, dtype=torch.float32, device=device)  # violations only
    pay_k = torch.empty((slab_blocks, bs, H, D), dtype=dtype, device=device)
    pay_v = torch.empty_like(pay_k)
    blkmap = torch.empty(P * L * nb, dtype=torch.int32, device=device)
    starts = np.concatenate([[0], np.cumsum(caps * L)[:-1]])
    blk_bytes = bs * H * D * pay_k.element_size()
    # descriptors (pairs, outputs) and the hinted-block mask in ONE upload
    desc = np.zeros(P * (_lib.DIFF_PAIR.itemsize + _lib.DIFF_OUT.itemsize) + P * nb, np.uint8)
    pairs = desc[:P * 32].view(_lib.DIFF_PAIR)
    outs = desc[P * 32:P * 72].view(_lib.DIFF_OUT)
    pairs["master_k"], pairs["master_v"] = ptr(mk), ptr(mv)
    pairs["mirror_k"] = [ptr(a) for a, _ in mirrors_dev]
    pairs["mirror_v"] = [ptr(b) for _, b in mirrors_dev]
    outs["payload_k"] = ptr(pay_k) + starts * blk_bytes
    outs["payload_v"] = ptr(pay_v) + starts * blk_bytes
    outs["indices"] = ptr(indices) + starts * 4
    outs["blkmap"] = ptr(blkmap) + np.arange(P, dtype=np.int64) * (L * nb * 4)
    outs["cap"] = caps
    desc[P * 72:] = hinted.reshape(-1)
    d_desc = upload(desc, device)
    d_pairs, d_outs, d_hinted = ptr(d_desc), ptr(d_desc) + P * 32, ptr(d_desc) + P * 72
    code = dtype_code(dtype)
    stream = stream_handle(device)
    if _SINGLE_PASS:
        # one launch: compare + look-back compaction + payload copy
        flags = torch.empty(P * L * nb + 1, dtype=torch.int32, device=device)
        _lib.call("tdkv_diff_encode", d_pairs, d_outs, P, d_hinted, ptr(flags),
                  ptr(flags) + 4 * P * L * nb, ptr(counts), ptr(violation), ptr(viol_maxabs),
                  L, total, H, D, bs, code, stream)
    else:
        _lib.call("tdkv_diff_compare", d_pairs, P, d_hinted, ptr(changed), ptr(violation),
                  ptr(viol_maxabs), L, total, H, D, bs, code, stream)
        _lib.call("tdkv_diff_compact", d_pairs, d_outs, P, ptr(changed), ptr(counts),
                  L, total, H, D, bs, code, stream)
    return _EncodeState(P, L, H, D, bs, nb, total, caps, starts, meta, viol_maxabs, pay_k,
                        pay_v, blkmap)


@dataclass
class _EncodeState:
    """Launched-but-unread encoder outputs (see encode_launch)."""

    P: int
    L: int
    H: int
    D: int
    bs: int
    nb: int
    total: int
    caps: np.ndarray
    starts: np.ndarray
    meta: torch.Tensor
    viol_maxabs: torch.Tensor
    pay_k: torch.Tensor
    pay_v: torch.Tensor
    blkmap: torch.Tensor


def encode_batch(master: LayeredKv, mirrors: Sequence[LayeredKv],
                 hint_positions: Sequence[np.ndarray], blocks: CacheBlockConfig,
                 device: Optional[torch.device] = None) -> List[BlockSparseDiff]:
    """Encode many mirrors against one master in one kernel launch (K2).

    Raises HintSoundnessError for the first mirror (in list order) that
    differs outside its hints, at that mirror's first (layer, block) in
    layer-major order -- the block encode_diff would raise on.
    """
    if len(mirrors) != len(hint_positions):
        raise ValueError("one hint array per mirror")
    if not mirrors:
        return []
    return encode_finish(encode_launch(master, mirrors, hint_positions, blocks, device))


def encode_finish(st: "_EncodeState") -> List[BlockSparseDiff]:
    """The one device->host read of an encode (violations, counts, indices)
    and the diffs as views of the device payload slab."""
    P, L, H, D, bs, nb, total = st.P, st.L, st.H, st.D, st.bs, st.nb, st.total
    caps, starts, meta, viol_maxabs = st.caps, st.starts, st.meta, st.viol_maxabs
    pay_k, pay_v, blkmap = st.pay_k, st.pay_v, st.blkmap
    meta_h = meta.cpu().numpy()
    viol_h = meta_h[:P]
    bad = np.flatnonzero(viol_h != _lib.NO_VIOLATION)
    if bad.size:
        p = int(bad[0])
        v = int(viol_h[p])
        layer, b = divmod(v, nb)
        worst = float(viol_maxabs[(p * L + layer) * nb + b].item())
        raise HintSoundnessError(
            f"layer {layer} block {b} differs outside the hinted positions (max abs {worst:.3e})")
    counts_h = meta_h[P:P + P * L].reshape(P, L)
    idx_h = meta_h[P + P * L:]
    diffs = []
    for p in range(P):
        s, cap = int(starts[p]), int(caps[p])
        slab = _EncodedSlab(counts_h[p], idx_h[s:s + L * cap], cap, pay_k, pay_v, s,
                            blkmap, p * L * nb, L * nb)
        diffs.append(BlockSparseDiff._from_slab(L, bs, H, D, total, slab))
    return diffs


def encode_diff(master: LayeredKv, mirror: LayeredKv, hint_positions: np.ndarray,
                blocks: CacheBlockConfig) -> BlockSparseDiff:
    """Block-sparse difference of mirror against master (diffstore.py:119-182).

    Host (numpy) inputs produce a diff with host numpy payloads; device
    inputs keep the payload on the device."""
    diff = encode_batch(master, [mirror], [hint_positions], blocks)[0]
    return diff if master.on_device else diff.to_host()


# ---------------------------------------------------------------------------
# dense decode (K3 with identity rows, no rotation)


def diff_decode_dense(master: LayeredKv, diff: BlockSparseDiff) -> LayeredKv:
    """Materialize the mirror's full planes: master + changed blocks."""
    if (master.num_layers != diff.num_layers or master.num_tokens != diff.total_tokens
            or tuple(master.k.shape[2:]) != (diff.num_heads, diff.head_dim)):
        raise ValueError("diff does not describe this master")
    device = master.k.device if master.on_device else default_device()
    dtype = _plane_dtype(master)
    mk = to_device(master.k, device, dtype)
    mv = to_device(master.v, device, dtype)
    out_k = torch.empty_like(mk)
    out_v = torch.empty_like(mv)
    decode_dense_into(mk, mv, diff, out_k, out_v)
    if master.on_device:
        return LayeredKv(out_k, out_v, master.positions.copy())
    return LayeredKv(to_host(out_k), to_host(out_v), master.positions.copy())


def decode_dense_into(mk: torch.Tensor, mv: torch.Tensor, diff: BlockSparseDiff,
                      out_k: torch.Tensor, out_v: torch.Tensor) -> None:
    L, T, H, D = mk.shape
    dd = diff.device_form(mk.device, mk.dtype)
    job = _kernels.rows_job(mk, mv, T * H * D, out_k, out_v, T * H * D, T, pay_k=dd.pay_k,
                            pay_v=dd.pay_v, map_k=dd.map_k, map_v=dd.map_v)
    _kernels.rows(_kernels.rows_jobs([job]), T, None, L, H, D, diff.block_size, mk.dtype,
                  mk.device)


# ---------------------------------------------------------------------------
# wire format (host)


def wire_nbytes(diff: BlockSparseDiff, itemsize: int = 4) -> int:
    """Serialized size without building the bytes: header, per layer
    count+flag+indices(+escape fields)+payload, trailer.  itemsize=4 is the
    reference's float32 wire (equal to len(serialize_diff(diff)))."""
    blk = diff.block_size * diff.num_heads * diff.head_dim * itemsize
    n = _HEADER.size + 4
    for kc, vc, escape in diff._plane_counts():
        n += 5 + 4 * kc + kc * blk + vc * blk
        if escape:
            n += 4 + 4 * vc
    return n


def _f32_bytes(x) -> bytes:
    if isinstance(x, torch.Tensor):
        x = to_host(x)
    return np.ascontiguousarray(x, dtype="<f4").tobytes()


def _serialize_host(diff: BlockSparseDiff) -> bytes:
    parts = [_HEADER.pack(MAGIC, VERSION, diff.num_layers, diff.block_size, diff.num_heads,
                          diff.head_dim, diff.total_tokens)]
    for ld in diff.layers:
        shared = ld.v_indices is None
        parts.append(struct.pack("<IB", ld.indices.size, 1 if shared else 0))
        parts.append(ld.indices.astype("<u4").tobytes())
        parts.append(_f32_bytes(ld.k_blocks))
        if not shared:
            parts.append(struct.pack("<I", ld.v_indices.size))
            parts.append(ld.v_indices.astype("<u4").tobytes())
        parts.append(_f32_bytes(ld.v_blocks))
    parts.append(struct.pack("<I", CacheBlockConfig(diff.block_size).valid_len(diff.total_tokens)))
    return b"".join(parts)


def _gpu_packable(diff: BlockSparseDiff) -> bool:
    """Encoder-produced diffs (payload in a device slab, shared K/V indices)
    are packed on the GPU; anything else takes the host path."""
    return diff._slab is not None and diff._slab.pay_k.is_cuda


def _pack_segments(diff: BlockSparseDiff, base: int, lit: bytearray, segs: list) -> int:
    """Append the wire segments of one slab-backed diff at image offset
    ``base``; literal bytes (header, counts, flags, indices, trailer) go to
    ``lit`` (uploaded once) and are referenced by their offset there.
    Returns the image length."""
    s = diff._slab
    pay_k, pay_v = s.pay_k, s.pay_v
    esz = pay_k.element_size()
    blk = diff.block_size * diff.num_heads * diff.head_dim
    kind = _lib.WIRE_BF16_TO_F32 if pay_k.dtype == torch.bfloat16 else _lib.WIRE_RAW
    off = base

    def literal(b: bytes) -> None:
        nonlocal off
        segs.append((off, len(b), -1 - len(lit), _lib.WIRE_RAW))   # negative = literal
        lit.extend(b)
        off += len(b)

    literal(_HEADER.pack(MAGIC, VERSION, diff.num_layers, diff.block_size, diff.num_heads,
                         diff.head_dim, diff.total_tokens))
    for layer in range(diff.num_layers):
        c = int(s.counts[layer])
        row0 = layer * s.cap
        idx = s.idx[row0:row0 + c].astype("<u4").tobytes()
        literal(struct.pack("<IB", c, 1) + idx)
        for plane in (pay_k, pay_v):
            if c:
                segs.append((off, c * blk * 4, ptr(plane) + row0 * blk * esz, kind))
                off += c * blk * 4
    literal(struct.pack("<I", CacheBlockConfig(diff.block_size).valid_len(diff.total_tokens)))
    return off - base


def serialize_many(diffs: Sequence[BlockSparseDiff], copy: bool = True) -> list:
    """Wire images of several diffs.  Encoder-produced (device) diffs are
    packed by one tdkv_wire_pack launch into one device buffer (payload
    converted to float32 on the fly) and read back with one copy; the
    bytes are identical to serialize_diff (diffstore.py:210-239).

    ``copy=False`` returns the GPU-packed images as read-only memoryviews
    of one pinned host buffer (no per-image bytes object: building Python
    bytes from a fresh buffer runs at ~2 GB/s, the PCIe read at ~50)."""
    out: list = [None] * len(diffs)
    gpu = [i for i, d in enumerate(diffs) if _gpu_packable(d)]
    for i, d in enumerate(diffs):
        if i not in gpu:
            out[i] = _serialize_host(d)
    if not gpu:
        return out
    device = diffs[gpu[0]]._slab.pay_k.device
    release_inflight()      # earlier direct H2Ds from pinned images that have drained
    lit = bytearray()
    segs: list = []
    spans = []
    base = 0
    for i in gpu:
        n = _pack_segments(diffs[i], base, lit, segs)
        spans.append((base, n))
        base += (n + 15) & ~15
    d_lit = upload(np.frombuffer(lit, np.uint8), device)
    table = np.zeros(len(segs), _lib.WIRE_SEG)
    for j, (o, n, p, k) in enumerate(segs):
        table[j] = (o, n, p if p >= 0 else ptr(d_lit) + (-1 - p), k, 0)
    d_table = upload(table.view(np.uint8), device)
    image = torch.empty(base + 16, dtype=torch.uint8, device=device)
    _lib.call("tdkv_wire_pack", ptr(d_table), len(segs), int(table["nbytes"].max()), ptr(image),
              stream_handle(device))
    host = torch.empty(base, dtype=torch.uint8, pin_memory=base >= 1 << 16)
    host.copy_(image[:base])
    buf = host.numpy()
    view = memoryview(buf).toreadonly()
    for i, (o, n) in zip(gpu, spans):
        out[i] = buf[o:o + n].tobytes() if copy else view[o:o + n]
    return out


def serialize_diff(diff: BlockSparseDiff) -> bytes:
    """The TDDF wire image (diffstore.py:210-239): GPU-packed for encoder
    output, host-assembled otherwise; byte-identical either way."""
    return serialize_many([diff])[0]


class _Cursor:
    def __init__(self, buf: bytes) -> None:
        self.buf = buf
        self.pos = 0

    def take(self, n: int, what: str) -> bytes:
        if self.pos + n > len(self.buf):
            raise MalformedDiffError(f"truncated diff: expected {what}")
        out = self.buf[self.pos:self.pos + n]
        self.pos += n
        return out

    def skip(self, n: int, what: str) -> int:
        if self.pos + n > len(self.buf):
            raise MalformedDiffError(f"truncated diff: expected {what}")
        at = self.pos
        self.pos += n
        return at

    def u32(self, what: str) -> int:
        return struct.unpack("<I", self.take(4, what))[0]

    def ids(self, count: int, what: str) -> np.ndarray:
        a = np.frombuffer(self.take(4 * count, what), dtype="<u4").astype(np.int64)
        if a.size > 1 and not (np.diff(a) > 0).all():
            raise MalformedDiffError(f"{what} must be strictly increasing")
        return a


@dataclass
class _WireLayer:
    indices: np.ndarray
    k_off: int                   # byte offset of the K payload in the image
    v_indices: Optional[np.ndarray]
    v_off: int


def _parse_wire(buf: bytes):
    """Structural parse + every check of deserialize_diff (diffstore.py:242-306)
    without touching the payload bytes: geometry and per-layer index arrays
    and payload offsets."""
    cur = _Cursor(buf)
    magic, version, num_layers, bs, heads, dim, total = _HEADER.unpack(
        cur.take(_HEADER.size, "header"))
    if magic != MAGIC:
        raise MalformedDiffError("bad magic")
    if version != VERSION:
        raise MalformedDiffError(f"unsupported version {version}")
    if min(num_layers, bs, heads, dim, total) <= 0:
        raise MalformedDiffError("non-positive geometry field")
    blk_bytes = bs * heads * dim * 4
    layers = []
    for layer in range(num_layers):
        count = cur.u32(f"layer {layer} count")
        flag = cur.take(1, f"layer {layer} index flag")[0]
        if flag not in (0, 1):
            raise MalformedDiffError(f"layer {layer}: unknown index flag {flag}")
        idx = cur.ids(count, f"layer {layer} indices")
        k_off = cur.skip(count * blk_bytes, f"layer {layer} K payload")
        if flag == 1:
            v_off = cur.skip(count * blk_bytes, f"layer {layer} V payload")
            layers.append(_WireLayer(idx, k_off, None, v_off))
        else:
            vc = cur.u32(f"layer {layer} V count")
            vidx = cur.ids(vc, f"layer {layer} V indices")
            v_off = cur.skip(vc * blk_bytes, f"layer {layer} V payload")
            layers.append(_WireLayer(idx, k_off, vidx, v_off))
    valid = cur.u32("valid_len trailer")
    if cur.pos != len(buf):
        raise MalformedDiffError("trailing bytes after diff")
    nb = CacheBlockConfig(bs).num_blocks(total)
    for wl in layers:
        for ids in (wl.indices, wl.v_indices):
            if ids is not None and ids.size and ids.max() >= nb:
                raise ValueError("block index out of range")
    if valid != CacheBlockConfig(bs).valid_len(total):
        raise MalformedDiffError("valid_len disagrees with token count")
    return (num_layers, bs, heads, dim, total), layers


def deserialize_diff(buf: bytes) -> BlockSparseDiff:
    """Parse a wire image into a host (numpy float32) diff (diffstore.py:242-306)."""
    (num_layers, bs, heads, dim, total), wls = _parse_wire(buf)
    shape = (bs, heads, dim)
    blk = bs * heads * dim

    def blocks(off: int, count: int) -> np.ndarray:
        return np.frombuffer(buf, dtype="<f4", count=count * blk, offset=off).astype(
            np.float32).reshape((count,) + shape)

    layers = []
    for wl in wls:
        vc = wl.indices.size if wl.v_indices is None else wl.v_indices.size
        layers.append(LayerDiff(wl.indices, blocks(wl.k_off, wl.indices.size),
                                blocks(wl.v_off, vc), v_indices=wl.v_indices))
    return BlockSparseDiff(num_layers, bs, heads, dim, total, layers)


def deserialize_to_device(buf: bytes, device: Optional[torch.device] = None,
                          dtype: torch.dtype = torch.bfloat16) -> BlockSparseDiff:
    """Parse a wire image straight into a device diff ready for the fused
    restore: the host validates the structure (same errors as
    deserialize_diff), the image crosses PCIe once and one tdkv_wire_unpack
    launch scatters every payload block into a K and a V slab (float32 wire
    -> ``dtype``); the block maps are built on the host from the indices."""
    device = device or default_device()
    (num_layers, bs, heads, dim, total), wls = _parse_wire(buf)
    nb = CacheBlockConfig(bs).num_blocks(total)
    blk = bs * heads * dim
    kc = [wl.indices.size for wl in wls]
    vc = [wl.indices.size if wl.v_indices is None else wl.v_indices.size for wl in wls]
    k_rows, v_rows = _excl(kc), _excl(vc)
    pay_k = torch.empty((max(1, sum(kc)), bs, heads, dim), dtype=dtype, device=device)
    pay_v = torch.empty((max(1, sum(vc)), bs, heads, dim), dtype=dtype, device=device)
    kind = _lib.WIRE_F32_TO_BF16 if dtype == torch.bfloat16 else _lib.WIRE_RAW
    esz = pay_k.element_size()
    maps = np.full((2, num_layers, nb), -1, np.int32)
    segs = []
    for layer, wl in enumerate(wls):
        vidx = wl.indices if wl.v_indices is None else wl.v_indices
        maps[0, layer, wl.indices] = k_rows[layer] + np.arange(kc[layer], dtype=np.int32)
        maps[1, layer, vidx] = v_rows[layer] + np.arange(vc[layer], dtype=np.int32)
        if kc[layer]:
            segs.append((wl.k_off, kc[layer] * blk * 4, ptr(pay_k) + k_rows[layer] * blk * esz,
                         kind, 0))
        if vc[layer]:
            segs.append((wl.v_off, vc[layer] * blk * 4, ptr(pay_v) + v_rows[layer] * blk * esz,
                         kind, 0))
    # the image (+ 4 bytes of padding for the funnel-shift reads) in one copy
    image = bytes_to_device(buf, device, pad=8)
    table = np.array(segs, dtype=_lib.WIRE_SEG) if segs else np.zeros(0, _lib.WIRE_SEG)
    d_maps = torch.from_numpy(maps.reshape(2, -1)).to(device, non_blocking=True)
    if segs:
        d_table = upload(table.view(np.uint8), device)
        _lib.call("tdkv_wire_unpack", ptr(d_table), len(segs), int(table["nbytes"].max()),
                  ptr(image), stream_handle(device))
    layers = []
    for layer, wl in enumerate(wls):
        k0, v0 = k_rows[layer], v_rows[layer]
        layers.append(LayerDiff(wl.indices, pay_k[k0:k0 + kc[layer]], pay_v[v0:v0 + vc[layer]],
                                v_indices=wl.v_indices))
    diff = BlockSparseDiff(num_layers, bs, heads, dim, total, layers)
    diff._dev = _DeviceDiff(pay_k, pay_v, d_maps[0], d_maps[1])
    diff._keepalive = image                       # until the unpack has run
    return diff


def _excl(counts) -> List[int]:
    out, acc = [], 0
    for c in counts:
        out.append(acc)
        acc += c
    return out


# ---------------------------------------------------------------------------
# families (diffstore.py:313-457)


@dataclass(eq=False)
class MasterEntry:
    family_id: int
    kv: LayeredKv
    tokens: Optional[tuple] = None
    pin_count: int = 0


@dataclass(eq=False)
class MirrorHandle:
    """Master reference + block-sparse diff; pins the master while live."""

    family_id: int
    request_id: int
    master: MasterEntry
    diff: BlockSparseDiff
    released: bool = field(default=False, init=False)

    @property
    def positions(self) -> np.ndarray:
        return self.master.kv.positions

    def release(self) -> None:
        if self.released:
            raise ValueError("mirror handle already released")
        self.released = True
        self.master.pin_count -= 1


@dataclass(eq=False)
class CompressionStats:
    dense_nbytes: int
    diff_payload_nbytes: List[int]
    diff_serialized_nbytes: List[int]
    changed_blocks: List[int]

    @property
    def ratios(self) -> List[float]:
        return [self.dense_nbytes / b for b in self.diff_serialized_nbytes]

    @property
    def family_cost(self) -> float:
        return 1.0 + sum(b / self.dense_nbytes for b in self.diff_serialized_nbytes)


def family_cost_from_ratio(num_members: int, ratio: float) -> float:
    if num_members < 1:
        raise ValueError("a family has at least one member")
    if ratio <= 0:
        raise ValueError("compression ratio must be positive")
    return 1.0 + (num_members - 1) / ratio


@dataclass(eq=False)
class FamilyEncoding:
    master: MasterEntry
    mirrors: Dict[int, MirrorHandle]
    stats: CompressionStats


class DiffStore:
    """Registry of cache families: dense masters and diff-encoded mirrors."""

    def __init__(self, blocks: CacheBlockConfig) -> None:
        self.blocks = blocks
        self._families: Dict[int, FamilyEncoding] = {}
        self._next_id = 0
        self._lock = threading.Lock()

    def __len__(self) -> int:
        return len(self._families)

    def register_dense(self, kv: LayeredKv, tokens: Optional[Sequence[int]] = None) -> MasterEntry:
        with self._lock:
            fid = self._next_id
            self._next_id += 1
            master = MasterEntry(fid, kv.copy(),
                                 None if tokens is None else tuple(int(t) for t in tokens))
            L, T, H, D = (int(x) for x in kv.k.shape)
            self._families[fid] = FamilyEncoding(
                master, {}, CompressionStats(kv_dense_nbytes(T, L, H, D), [], [], []))
            return master

    def encode_family(self, plan, results, tokens: Optional[Sequence[int]] = None) -> FamilyEncoding:
        """Master stays dense; every other member becomes a diff against it.
        All mirrors are encoded in one batched K2 pass (ascending rid order)."""
        master_kv = results[plan.master_id].kv
        items = sorted(plan.mirror_diff_hints.items())
        mirrors_kv = [results[rid].kv for rid, _ in items]
        diffs = encode_batch(master_kv, mirrors_kv, [h for _, h in items], self.blocks)
        if not master_kv.on_device:
            diffs = [d.to_host() for d in diffs]
        master = self.register_dense(master_kv, tokens)
        # wire sizes are those of the image serialize_diff emits: the
        # reference's float32 TDDF for every dtype (diffstore.py:431 measures
        # len(serialize_diff(d))); wire_nbytes(d) == len(serialize_diff(d))
        mirrors, payload, wire, changed = {}, [], [], []
        diff_f32 = _plane_dtype(master_kv) == torch.float32
        for (rid, _), diff in zip(items, diffs):
            mirrors[rid] = MirrorHandle(master.family_id, rid, master, diff)
            master.pin_count += 1
            # float32 payload bytes (== diff.payload_nbytes for float32 planes)
            payload.append(diff.payload_nbytes if diff_f32 else
                           2 * 4 * diff.block_size * diff.num_heads * diff.head_dim
                           * sum(diff.changed_blocks_per_layer))
            wire.append(wire_nbytes(diff))
            changed.append(sum(diff.changed_blocks_per_layer))
        # dense bytes as the reference defines them (float32 K+V, core.py:33-35
        # and CompressionStats, diffstore.py:349-366), so ratios and
        # family_cost compare float32 dense with the float32 wire for every
        # plane dtype -- the figures the reference reports on the f32-upcast
        # cache
        L, T, H, D = (int(x) for x in master_kv.k.shape)
        enc = FamilyEncoding(master, mirrors,
                             CompressionStats(kv_dense_nbytes(T, L, H, D), payload, wire, changed))
        with self._lock:
            self._families[master.family_id] = enc
        return enc

    def family(self, family_id: int) -> FamilyEncoding:
        with self._lock:
            return self._families[family_id]

    def drop_family(self, family_id: int) -> None:
        with self._lock:
            enc = self._families[family_id]
            if enc.master.pin_count > 0:
                raise PinnedMasterError(
                    f"family {family_id} has {enc.master.pin_count} live mirrors")
            del self._families[family_id]

    def is_pinned(self, ref: object) -> bool:
        return isinstance(ref, MasterEntry) and ref.pin_count > 0
