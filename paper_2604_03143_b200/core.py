"""Value types of the hot path (reference: roundkv/core.py).

``LayeredKv`` (core.py:164-201), ``PositionSpan`` (core.py:204-237),
``CacheBlockConfig`` (core.py:240-263) and the toy model's ``ModelConfig``
(core.py:38-66) keep the reference's constructors, validation and error
messages.  KV planes may be host numpy float32 arrays
(the reference's contract) or CUDA tensors in float32 or bfloat16 (the
B200-resident form); positions are always host int64 metadata.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

import numpy as np
import torch


def kv_dense_nbytes(num_tokens: int, num_layers: int, num_heads: int, head_dim: int,
                    itemsize: int = 4) -> int:
    """Bytes of a dense K+V cache (core.py:33-35; float32 unless told)."""
    return num_tokens * num_layers * num_heads * head_dim * 2 * itemsize


def union_sorted(*arrays) -> np.ndarray:
    """np.union1d of int arrays as int64 (sorted, unique) by one sort and an
    adjacent-difference mask -- several times cheaper than union1d's hashing
    unique for the short index vectors of a recovery round."""
    c = np.concatenate([np.asarray(a, np.int64).reshape(-1) for a in arrays])
    if c.size < 2:
        return c
    c.sort()
    keep = np.empty(c.size, bool)
    keep[0] = True
    np.not_equal(c[1:], c[:-1], out=keep[1:])
    return c[keep]


def _strictly_increasing(a: np.ndarray) -> bool:
    return a.size < 2 or bool((a[1:] > a[:-1]).all())


def plane_nbytes(x) -> int:
    if isinstance(x, torch.Tensor):
        return x.numel() * x.element_size()
    return int(x.nbytes)


def _plane_ok(x) -> bool:
    if isinstance(x, np.ndarray):
        return x.dtype == np.float32
    if isinstance(x, torch.Tensor):
        return x.dtype in (torch.float32, torch.bfloat16) and x.device.type == "cuda"
    return False


@dataclass(eq=False)
class LayeredKv:
    """(L, T, H, D) K and V planes plus the absolute positions K encodes."""

    k: object
    v: object
    positions: np.ndarray

    def __post_init__(self) -> None:
        if tuple(self.k.shape) != tuple(self.v.shape) or len(self.k.shape) != 4:
            raise ValueError("k and v must share a (L, T, H, D) shape")
        if not (_plane_ok(self.k) and _plane_ok(self.v)) or type(self.k) is not type(self.v):
            raise ValueError("kv tensors must be float32")
        if isinstance(self.k, torch.Tensor) and self.k.dtype != self.v.dtype:
            raise ValueError("k and v must share a dtype")
        self.positions = np.asarray(self.positions, dtype=np.int64)
        if self.positions.shape != (self.k.shape[1],):
            raise ValueError("positions must have one entry per token")
        if not _strictly_increasing(self.positions):
            raise ValueError("positions must be strictly increasing")

    @property
    def num_layers(self) -> int:
        return int(self.k.shape[0])

    @property
    def num_tokens(self) -> int:
        return int(self.k.shape[1])

    @property
    def num_heads(self) -> int:
        return int(self.k.shape[2])

    @property
    def head_dim(self) -> int:
        return int(self.k.shape[3])

    @property
    def on_device(self) -> bool:
        return isinstance(self.k, torch.Tensor)

    @property
    def dense_nbytes(self) -> int:
        return plane_nbytes(self.k) + plane_nbytes(self.v)

    def copy(self) -> "LayeredKv":
        if self.on_device:
            return LayeredKv(self.k.clone(), self.v.clone(), self.positions.copy())
        return LayeredKv(self.k.copy(), self.v.copy(), self.positions.copy())


@dataclass(frozen=True, eq=False)
class PositionSpan:
    """Mapping from the positions rows were computed at to new positions."""

    old_positions: np.ndarray
    new_positions: np.ndarray

    def __post_init__(self) -> None:
        old = np.asarray(self.old_positions, dtype=np.int64)
        new = np.asarray(self.new_positions, dtype=np.int64)
        if old.shape != new.shape or old.ndim != 1:
            raise ValueError("old and new positions must be 1-d and equal length")
        if not (_strictly_increasing(old) and _strictly_increasing(new)):
            raise ValueError("span positions must be strictly increasing")
        object.__setattr__(self, "old_positions", old)
        object.__setattr__(self, "new_positions", new)
        object.__setattr__(self, "_delta", None)

    def __len__(self) -> int:
        return int(self.old_positions.size)

    @property
    def delta(self) -> np.ndarray:
        """new - old (computed once: a span is immutable; read-only view)."""
        d = self._delta
        if d is None:
            d = self.new_positions - self.old_positions
            d.flags.writeable = False
            object.__setattr__(self, "_delta", d)
        return d

    @classmethod
    def identity(cls, positions: Iterable[int]) -> "PositionSpan":
        pos = np.fromiter((int(p) for p in positions), dtype=np.int64)
        return cls(pos, pos.copy())

    @classmethod
    def shifted(cls, positions: Iterable[int], offset: int) -> "PositionSpan":
        pos = np.fromiter((int(p) for p in positions), dtype=np.int64)
        return cls(pos, pos + int(offset))


@dataclass(frozen=True)
class CacheBlockConfig:
    """Token-block geometry shared by the pool, the diff codec and restores."""

    block_size: int = 32

    def __post_init__(self) -> None:
        if self.block_size < 1:
            raise ValueError("block_size must be positive")

    def num_blocks(self, num_tokens: int) -> int:
        return (num_tokens + self.block_size - 1) // self.block_size

    def block_bounds(self, block: int, num_tokens: int) -> tuple:
        lo = block * self.block_size
        if lo >= num_tokens:
            raise ValueError("block index out of range")
        return lo, min(lo + self.block_size, num_tokens)

    def valid_len(self, num_tokens: int) -> int:
        rem = num_tokens % self.block_size
        return rem if rem else min(self.block_size, num_tokens)


@dataclass(frozen=True)
class ModelConfig:
    """Dimensions and seeds of the deterministic toy transformer (core.py:38-66)."""

    num_layers: int = 4
    num_heads: int = 2
    head_dim: int = 8
    vocab_size: int = 1024
    rope_base: float = 10000.0
    weight_seed: int = 0

    def __post_init__(self) -> None:
        if self.num_layers < 1 or self.num_heads < 1:
            raise ValueError("num_layers and num_heads must be positive")
        if self.head_dim < 2 or self.head_dim % 2 != 0:
            raise ValueError("head_dim must be a positive even integer")
        if self.vocab_size < 2:
            raise ValueError("vocab_size must leave room for the separator id")
        if self.rope_base <= 0:
            raise ValueError("rope_base must be positive")

    @property
    def hidden_dim(self) -> int:
        return self.num_heads * self.head_dim

    @property
    def separator_token(self) -> int:
        # the highest id is reserved (the reference's workload draws below it)
        return self.vocab_size - 1
