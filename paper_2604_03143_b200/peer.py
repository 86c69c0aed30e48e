"""The All-Gather exchange fused into the collector: K1 reads master tiles
from the producing GPU over NVLink.

In an All-Gather round every agent's output block becomes a shared segment
master on the GPU that ran the agent.  The NCCL form (``dist.broadcast_collect``)
first copies every master into each rank's own arena, then collects from it.
Here each rank instead maps its peers' arenas into its address space once
(CUDA IPC through torch's tensor sharing), and one ``tdkv_collect_sources``
launch per round stages every master tile straight from its owner's HBM into
shared memory with the TMA engine, rotates K and scatters K/V into the local
pool.  No received copy of the masters is written to local HBM, no chunking
or per-chunk synchronization is needed, and each owner serves each master
byte once per reader, spread over the whole kernel.

Round protocol (``PeerRound``): owners finish writing their masters, all
ranks meet at a barrier (``ready``), every rank collects, and all ranks meet
again (``done``) before an owner may overwrite its masters for the next round.

Reference: the reference keeps every master in one process (trace.py:161-184)
and collects with align_cached (pic.py:208-235) + the _skeleton V copy
(pic.py:203-204) + write_rows (paged_pool.py:150-156).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist
from torch.multiprocessing.reductions import reduce_tensor

from .collector import CollectPlan, MasterArena
from ._device import upload


def contiguous_owners(num_segments: int, world: int) -> np.ndarray:
    """Owner rank of each segment when segments are produced by contiguous
    agent shards: segment s on rank floor(s * world / S)."""
    return (np.arange(num_segments, dtype=np.int64) * world // max(1, num_segments)).astype(
        np.int64)


def open_peer_arenas(arena: MasterArena, group=None) -> List[MasterArena]:
    """Every rank's arena as seen from this rank: the local one for this rank,
    the peers' mapped by CUDA IPC (their device memory, reached over NVLink
    when the ranks sit on different GPUs).  Collective: all ranks call it.
    Every arena must have the same layout."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    mine = (reduce_tensor(arena.k), reduce_tensor(arena.v), tuple(arena.k.shape),
            str(arena.k.dtype))
    everyone: list = [None] * world
    dist.all_gather_object(everyone, mine, group=group)
    out = []
    for r, (kh, vh, shape, dtype) in enumerate(everyone):
        if shape != tuple(arena.k.shape) or dtype != str(arena.k.dtype):
            raise ValueError(f"rank {r}'s arena layout differs from rank {rank}'s")
        if r == rank:
            out.append(arena)
            continue
        k = kh[0](*kh[1])
        v = vh[0](*vh[1])
        out.append(MasterArena(k, v, arena.seg_row0, arena.seg_len, arena.source_positions))
    return out


class PeerRound:
    """One rank's side of peer-read rounds: ``collect(plan)`` runs K0 + one
    multi-source K1 over the plan, every unit's tile read from the arena of
    the rank that owns its segment."""

    def __init__(self, collector, seg_owner: Sequence[int], group=None) -> None:
        self.collector = collector
        self.group = group
        self.seg_owner = np.asarray(seg_owner, np.int64)
        if self.seg_owner.size != collector.arena.num_segments:
            raise ValueError("one owner per segment")
        self.sources = open_peer_arenas(collector.arena, group)
        if self.seg_owner.size and (self.seg_owner.min() < 0
                                    or self.seg_owner.max() >= len(self.sources)):
            raise ValueError("segment owner out of range")
        self._unit_src = {}
        self._flag = None

    def unit_sources(self, plan: CollectPlan) -> torch.Tensor:
        key = id(plan)
        hit = self._unit_src.get(key)
        if hit is None or hit[0] is not plan:
            arena = self.collector.arena
            src = plan.unit_sources(self.seg_owner, arena.seg_row0, arena.seg_len)
            hit = (plan, upload(np.ascontiguousarray(src), plan.device))
            self._unit_src[key] = hit
        return hit[1]

    def _sync(self) -> None:
        # NCCL: a one-element all-reduce queued on the current stream is a
        # device-side barrier -- it completes on a rank only once every rank's
        # stream has reached it, and the work queued after it waits for it --
        # so the host never blocks.  gloo (ranks sharing one GPU in the tests):
        # drain the device, then a host barrier.
        device = self.collector.pool.device
        if dist.get_backend(self.group) == "nccl":
            if self._flag is None:
                self._flag = torch.zeros(1, dtype=torch.int32, device=device)
            dist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.current_stream(device).synchronize()
            dist.barrier(group=self.group)

    def ready(self) -> None:
        """This round's masters are written on every owner (stream order):
        K1 launched after this may read them."""
        self._sync()

    def done(self) -> None:
        """Every rank has finished reading this round's masters: owners may
        overwrite them with work queued after this."""
        self._sync()

    def collect(self, plan: CollectPlan, ledger=None, grid_limit: int = 0) -> int:
        """K0 + K1 for ``plan`` (no barriers: call ``ready`` before and
        ``done`` after when the owners rewrite their masters between rounds)."""
        pool = self.collector.pool
        n = plan.launch_table()
        n += plan.launch_collect_sources(self.sources, self.unit_sources(plan), pool.k, pool.v,
                                         pool.layer_stride, grid_limit)
        if ledger is not None and plan.num_jobs:
            for layer in range(plan.num_layers):
                ledger.record_rope_call(layer)
        return n

    def round(self, plan: CollectPlan, ledger=None) -> int:
        """ready -> collect -> done."""
        self.ready()
        n = self.collect(plan, ledger)
        self.done()
        return n

    def peer_bytes(self, plan: CollectPlan, rank: Optional[int] = None) -> int:
        """Master bytes this rank reads from other ranks per round (each unit
        tile once per layer and plane)."""
        rank = dist.get_rank(self.group) if rank is None else rank
        arena = self.collector.arena
        src = plan.unit_sources(self.seg_owner, arena.seg_row0, arena.seg_len)
        rows = plan.units_host["nrows"].astype(np.int64)
        # units of one tile share rows: count each (row0) once
        foreign = src != rank
        tiles = {int(r0): int(n) for r0, n, f in zip(plan.units_host["row0"], rows, foreign) if f}
        row_bytes = int(arena.k.shape[2] * arena.k.shape[3]) * arena.k.element_size()
        return 2 * arena.num_layers * row_bytes * sum(tiles.values())
