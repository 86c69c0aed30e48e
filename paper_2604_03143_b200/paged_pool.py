"""Device-resident token-slot paged KV pool (reference: roundkv/paged_pool.py).

Layout is the reference's: one K and one V plane of shape
(num_layers, capacity, num_heads, head_dim) -- here in HBM, float32 or
bfloat16.  A slot addresses one token's row in every layer, so each
(layer, slot) row is H*D contiguous elements (1-2 KiB at Qwen2.5 shapes) and
any slot order stores fully coalesced.

The allocator keeps the reference policy exactly (paged_pool.py:106-135):
whole free blocks in ascending order first, then the lowest scattered free
slots -- in native code over free-slot / whole-block bitmaps
(``tdkv_alloc_*``), so slot maps are bit-identical to the reference's
without its O(capacity) Python loop.  ``choose_slots`` is the same policy in
numpy, kept as an executable statement of it for the host-side tests.  Slot maps are host
metadata; their device copies are cached on the SlotMap.
"""
from __future__ import annotations

import threading
from typing import Optional, Sequence

import numpy as np
import torch

from . import _kernels
from ._device import default_device, h2d, to_device, to_host


class OutOfSlotsError(RuntimeError):
    def __init__(self, requested: int, available: int) -> None:
        super().__init__(f"requested {requested} slots, {available} free")
        self.requested = requested
        self.available = available


class UseAfterFreeError(RuntimeError):
    """A slot was read after free (or before it was ever written)."""


class SlotMap:
    """Slots of one request in token order (paged_pool.py:29-48)."""

    __slots__ = ("request_id", "slots", "serial", "_dev", "lo", "hi")

    def __init__(self, request_id: int, slots, serial: int = -1) -> None:
        arr = np.asarray(slots, dtype=np.int64).reshape(-1)
        if np.unique(arr).size != arr.size:
            raise ValueError("slot map must not repeat slots")
        self.request_id = int(request_id)
        self.slots = arr
        self.serial = int(serial)
        self._dev = None
        # slot range, checked against a pool's capacity before any kernel
        # writes through the map (numpy's IndexError in the reference)
        self.lo = int(arr.min()) if arr.size else 0
        self.hi = int(arr.max()) if arr.size else -1

    def __len__(self) -> int:
        return int(self.slots.size)

    def device_slots(self, device: torch.device) -> torch.Tensor:
        d = self._dev
        if d is None or d.device != device:
            d = h2d(self.slots, device)
            self._dev = d
        return d


def slot_maps_disjoint(maps: Sequence[SlotMap]) -> bool:
    if not maps:
        return True
    cat = np.concatenate([m.slots for m in maps])
    return np.unique(cat).size == cat.size


def choose_slots(free: np.ndarray, num_tokens: int, block_size: int) -> np.ndarray:
    """Reference allocation policy over a boolean free mask (not mutated)."""
    cap = free.size
    nblk = (cap + block_size - 1) // block_size
    padded = np.ones(nblk * block_size, dtype=bool)
    padded[:cap] = free
    whole = np.flatnonzero(padded.reshape(nblk, block_size).all(axis=1))
    lens = np.minimum(block_size, cap - whole * block_size)
    parts = []
    need = num_tokens
    if whole.size:
        cum = np.cumsum(lens)
        k = int(np.searchsorted(cum, need))       # blocks [0, k] cover ``need``
        k = min(k, whole.size - 1)
        starts = whole[: k + 1] * block_size
        take = lens[: k + 1].copy()
        over = int(cum[k]) - need
        if over > 0:
            take[-1] -= over
        parts.append(np.repeat(starts, take) + (np.arange(int(take.sum()))
                                                - np.repeat(np.cumsum(take) - take, take)))
        need -= int(take.sum())
    if need > 0:
        mask = free.copy()
        if parts:
            mask[parts[0]] = False
        parts.append(np.flatnonzero(mask)[:need])
    return np.concatenate(parts).astype(np.int64) if parts else np.empty(0, np.int64)


class SlotAllocator:
    """The native (C++) slot allocator behind PagedPool: the reference policy
    (paged_pool.py:106-135) over free-slot / whole-block bitmaps."""

    def __init__(self, capacity: int, block_size: int) -> None:
        import ctypes
        from . import _lib
        self._lib = _lib.load()
        self._ct = ctypes
        self._h = self._lib.tdkv_alloc_create(int(capacity), int(block_size))
        if not self._h:
            raise ValueError(self._lib.tdkv_last_error().decode())

    def __del__(self) -> None:
        h = getattr(self, "_h", None)
        if h:
            self._lib.tdkv_alloc_destroy(h)
            self._h = None

    @property
    def free_count(self) -> int:
        return int(self._lib.tdkv_alloc_free_count(self._h))

    def take(self, n: int) -> np.ndarray:
        out = np.empty(int(n), dtype=np.int64)
        rc = self._lib.tdkv_alloc_take(self._h, int(n), out.ctypes.data_as(self._ct.c_void_p))
        if rc == 4:
            raise OutOfSlotsError(int(n), self.free_count)
        if rc:
            raise ValueError(self._lib.tdkv_last_error().decode())
        return out

    def release(self, slots: np.ndarray) -> None:
        s = np.ascontiguousarray(slots, dtype=np.int64)
        rc = self._lib.tdkv_alloc_release(self._h, s.ctypes.data_as(self._ct.c_void_p), s.size)
        if rc:
            raise ValueError(self._lib.tdkv_last_error().decode())


class PagedPool:
    """Fixed-capacity slot pool with per-layer K and V planes in HBM."""

    def __init__(self, capacity_tokens: int, num_layers: int, num_heads: int, head_dim: int,
                 block_size: int = 32, debug: bool = True, dtype: torch.dtype = torch.float32,
                 device: Optional[torch.device] = None) -> None:
        if capacity_tokens < 1:
            raise ValueError("capacity must be positive")
        self.capacity = int(capacity_tokens)
        self.block_size = int(block_size)
        self.debug = debug
        self.device = device or default_device()
        shape = (num_layers, self.capacity, num_heads, head_dim)
        self.k = torch.zeros(shape, dtype=dtype, device=self.device)
        self.v = torch.zeros(shape, dtype=dtype, device=self.device)
        self._alloc = SlotAllocator(self.capacity, self.block_size)
        self._nfree = self.capacity
        self._written = np.zeros((num_layers, self.capacity), dtype=bool)
        self._peak = 0
        self._next_serial = 0
        self._live: set = set()
        self._lock = threading.Lock()

    # -- geometry -----------------------------------------------------------
    @property
    def num_layers(self) -> int:
        return int(self.k.shape[0])

    @property
    def num_heads(self) -> int:
        return int(self.k.shape[2])

    @property
    def head_dim(self) -> int:
        return int(self.k.shape[3])

    @property
    def dtype(self) -> torch.dtype:
        return self.k.dtype

    @property
    def layer_stride(self) -> int:
        return self.capacity * self.num_heads * self.head_dim

    @property
    def free_count(self) -> int:
        return self._nfree

    @property
    def allocated_count(self) -> int:
        return self.capacity - self._nfree

    @property
    def peak_allocated(self) -> int:
        return self._peak

    def reset_peak(self) -> None:
        with self._lock:
            self._peak = self.allocated_count

    # -- allocator (host metadata) ------------------------------------------
    def allocate(self, num_tokens: int, request_id: int = 0) -> SlotMap:
        """Take ``num_tokens`` distinct slots, preferring whole free blocks."""
        if num_tokens < 1:
            raise ValueError("allocation must cover at least one token")
        with self._lock:
            if num_tokens > self._nfree:
                raise OutOfSlotsError(num_tokens, self._nfree)
            chosen = self._alloc.take(num_tokens)
            self._nfree -= chosen.size
            self._written[:, chosen] = False
            self._peak = max(self._peak, self.allocated_count)
            serial = self._next_serial
            self._next_serial += 1
            self._live.add(serial)
            return SlotMap(request_id, chosen, serial)

    def free(self, slot_map: SlotMap) -> None:
        """Return slots to the free list; debug mode poisons them with NaN."""
        with self._lock:
            if slot_map.serial not in self._live:
                raise ValueError("not a live allocation (double or foreign free)")
            self._live.discard(slot_map.serial)
            slots = slot_map.slots
            if self.debug and slots.size:
                rows = slot_map.device_slots(self.device)
                _kernels.fill_rows(self.k, rows, float("nan"))
                _kernels.fill_rows(self.v, rows, float("nan"))
            self._written[:, slots] = False
            self._alloc.release(slots)
            self._nfree += slots.size

    def mark_written(self, slot_map: SlotMap, layers: Optional[Sequence[int]] = None,
                     token_idx: Optional[np.ndarray] = None) -> None:
        """Record device-side writes (collector / restore kernels); the
        written map is only consulted by debug-mode reads."""
        if not self.debug:
            return
        slots = slot_map.slots if token_idx is None else slot_map.slots[token_idx]
        if layers is None:
            self._written[:, slots] = True
        else:
            self._written[np.asarray(layers)[:, None], slots[None, :]] = True

    # -- geometry checks before any kernel touches the planes ----------------
    def check_slots(self, slot_map: SlotMap) -> None:
        """Every slot of the map addresses a row of this pool (the kernels
        index the planes by slot without bounds checks)."""
        if slot_map.lo < 0 or slot_map.hi >= self.capacity:
            raise IndexError(f"slot map addresses slots [{slot_map.lo}, {slot_map.hi}] outside "
                             f"a pool of capacity {self.capacity}")

    def check_layer(self, layer: int) -> None:
        # numpy plane indexing: -L <= layer < L
        if not -self.num_layers <= int(layer) < self.num_layers:
            raise IndexError(f"layer {layer} out of range for {self.num_layers} layers")

    # -- row movement (K3) --------------------------------------------------
    def write_rows(self, slot_map: SlotMap, layer: int, k_rows, v_rows) -> None:
        slots = slot_map.slots
        if k_rows.shape[0] != slots.size or v_rows.shape[0] != slots.size:
            raise ValueError("row count must match the slot map")
        self.check_layer(layer)
        self.check_slots(slot_map)
        n = slots.size
        if n:
            kd = to_device(k_rows, self.device, self.dtype)
            vd = to_device(v_rows, self.device, self.dtype)
            H, D = self.num_heads, self.head_dim
            if tuple(kd.shape[1:]) != (H, D) or tuple(vd.shape[1:]) != (H, D):
                raise ValueError("rows must be (T, heads, head_dim)")
            job = _kernels.rows_job(kd, vd, 0, self.k[layer], self.v[layer], 0, n,
                                    dst_rows=slot_map.device_slots(self.device))
            _kernels.rows(_kernels.rows_jobs([job]), n, None, 1, H, D, _kernels.ROWS_BLOCK,
                          self.dtype, self.device)
        self._written[layer, slots] = True

    def read_rows(self, slot_map: SlotMap, layer: int, host: bool = True):
        """Gather one layer's rows for the slot map: numpy copies like the
        reference (paged_pool.py:158-164), or device tensors with host=False
        (the HBM-resident form, ``read_rows_device``)."""
        slots = slot_map.slots
        self.check_layer(layer)
        self.check_slots(slot_map)
        if self.debug and not self._written[layer, slots].all():
            raise UseAfterFreeError(f"layer {layer}: some slots were freed or never written")
        n = slots.size
        H, D = self.num_heads, self.head_dim
        k = torch.empty((n, H, D), dtype=self.dtype, device=self.device)
        v = torch.empty_like(k)
        if n:
            job = _kernels.rows_job(self.k[layer], self.v[layer], 0, k, v, 0, n,
                                    src_rows=slot_map.device_slots(self.device))
            _kernels.rows(_kernels.rows_jobs([job]), n, None, 1, H, D, _kernels.ROWS_BLOCK,
                          self.dtype, self.device)
        if host:
            return to_host(k), to_host(v)
        return k, v

    def read_rows_device(self, slot_map: SlotMap, layer: int):
        """read_rows with the rows left in HBM (device tensors)."""
        return self.read_rows(slot_map, layer, host=False)

    def check_conservation(self) -> None:
        assert 0 <= self._nfree <= self.capacity
        assert self._alloc.free_count == self._nfree
        assert self.allocated_count + self.free_count == self.capacity
