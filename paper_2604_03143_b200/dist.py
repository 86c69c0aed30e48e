"""Agent sharding across GPUs.

One process per GPU (``torch.distributed``, NCCL over NVLink on the B200
box, gloo for the CPU tests).  Agents are independent for the collector and
for mirror encoding, so each rank owns a contiguous agent range; the round
has two exchange steps:

* ``broadcast_arena`` -- the shared master blocks, once per round, from the
  rank that holds them (NCCL broadcast; every rank then runs K0 + K1 for its
  own agents);
* ``exchange_collect`` -- multi-session rounds sharded by agent
  (strong scaling): each session's masters live on the rank that runs the
  session's first agent and travel point-to-point (NCCL send/recv over
  NVLink) only to the other ranks whose shard touches that session, layer
  chunk by layer chunk, overlapped with K1 like ``broadcast_collect``;
* ``elect_master`` -- an all-gather of every rank's (deviation, request id)
  pairs so all ranks elect the same family master,
  argmin over (score, id) exactly as collective.select_master
  (collective.py:117-121);
* ``exchange_family_master`` / ``encode_family_sharded`` -- the family
  master cache (SURVEY §8e collective 3): the elected master's dense K/V
  planes go point-to-point from the rank holding them to every rank holding
  another member of the family, and each rank encodes its own mirrors against
  that one master (DiffStore.encode_family, diffstore.py:411-439: every
  mirror of a family is a diff against the same elected master).
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def shard_range(num_agents: int, rank: int, world: int) -> range:
    """Contiguous agent ids of ``rank``; shard sizes differ by at most one."""
    lo = rank * num_agents // world
    return range(lo, (rank + 1) * num_agents // world)


def broadcast_arena(arena, src: int = 0, group=None) -> int:
    """Broadcast the master arena's K and V planes from ``src``; returns the
    bytes each receiver gets."""
    dist.broadcast(arena.k, src, group=group)
    dist.broadcast(arena.v, src, group=group)
    return 2 * arena.k.numel() * arena.k.element_size()


def broadcast_collect(collector, plan, src: int = 0, chunks: int = 7, group=None,
                      ledger=None) -> int:
    """One round on one rank: the master arena arrives from ``src`` in layer
    chunks (NCCL broadcasts queued back to back on the communicator's
    stream) and K1 runs on each chunk as soon as it has landed, so the
    NVLink transfer of chunk c+1 overlaps the HBM-bound collector on chunk
    c.  ``plan`` may be a list (a rank's pool sub-batches).  Returns the
    kernels launched."""
    arena = collector.arena
    L = arena.num_layers
    plans = plan if isinstance(plan, (list, tuple)) else [plan]
    works = []
    for l0, l1 in _layer_chunks(L, chunks):
        wk = dist.broadcast(arena.k[l0:l1], src, group=group, async_op=True)
        wv = dist.broadcast(arena.v[l0:l1], src, group=group, async_op=True)
        works.append((l0, l1, wk, wv))
    pool = collector.pool
    n = sum(p.launch_table() for p in plans)
    for l0, l1, wk, wv in works:
        wk.wait()          # stream dependency for NCCL (host-blocking for gloo)
        wv.wait()
        for p in plans:
            n += p.launch_collect(arena, pool.k, pool.v, pool.layer_stride, layers=(l0, l1))
    if ledger is not None and any(p.num_jobs for p in plans):
        for layer in range(L):
            ledger.record_rope_call(layer)
    return n


def _layer_chunks(L: int, chunks: int):
    bounds = [round(i * L / chunks) for i in range(chunks + 1)]
    return [(l0, l1) for l0, l1 in zip(bounds[:-1], bounds[1:]) if l1 > l0]


def session_transfers(owners, needs):
    """(session, src, dst) for every rank that needs a session it does not
    own -- the round's whole exchange."""
    return [(s, owners[s], r) for r, ss in enumerate(needs) for s in ss if owners[s] != r]


class _StagedRecv:
    """A gloo receive of a CUDA tensor: lands in host memory, copied to the
    device on wait() (gloo point-to-point moves CPU tensors only; NCCL moves
    device memory directly)."""

    def __init__(self, work, host: torch.Tensor, dst: torch.Tensor) -> None:
        self.work, self.host, self.dst = work, host, dst

    def wait(self) -> None:
        self.work.wait()
        self.dst.copy_(self.host)


def exchange_sessions(arena, session_rows, transfers, rank: int, layers=None, group=None):
    """Post the point-to-point transfers of ``layers`` (default: all) of the
    sessions in ``transfers``; returns the requests to wait on (empty if this
    rank takes no part).  One op per (layer, plane, transfer): a layer's
    session rows are contiguous in the (L, rows, H, D) arena."""
    l0, l1 = layers or (0, arena.num_layers)
    staged = dist.get_backend(group) == "gloo" and arena.k.is_cuda
    ops, fixups = [], []
    for s, src, dst in transfers:
        if rank not in (src, dst):
            continue
        r0, r1 = session_rows[s]
        for layer in range(l0, l1):
            for plane in (arena.k, arena.v):
                t = plane[layer, r0:r1]
                if rank == src:
                    ops.append(dist.P2POp(dist.isend, t.cpu() if staged else t, dst, group=group))
                else:
                    buf = torch.empty(t.shape, dtype=t.dtype) if staged else t
                    ops.append(dist.P2POp(dist.irecv, buf, src, group=group))
                    if staged:
                        fixups.append((len(ops) - 1, buf, t))
    if not ops:
        return []
    reqs = list(dist.batch_isend_irecv(ops))
    for i, buf, t in fixups:
        reqs[i] = _StagedRecv(reqs[i], buf, t)
    return reqs


def exchange_collect(collector, plans, session_rows, transfers, rank: int, chunks: int = 4,
                     group=None) -> int:
    """One multi-session round on one rank: K0 for every plan, then per layer
    chunk the chunk's session transfers (send or receive) and K1 for the
    plans once the chunk has landed.  ``plans`` are this rank's sub-batches.
    Returns the kernels launched."""
    arena, pool = collector.arena, collector.pool
    n = sum(p.launch_table() for p in plans)
    pending = [(l0, l1, exchange_sessions(arena, session_rows, transfers, rank, (l0, l1), group))
               for l0, l1 in _layer_chunks(arena.num_layers, chunks)]
    for l0, l1, reqs in pending:
        for r in reqs:
            r.wait()
        for p in plans:
            n += p.launch_collect(arena, pool.k, pool.v, pool.layer_stride, layers=(l0, l1))
    return n


def elect_master(local_scores: Dict[int, float], group=None,
                 device: Optional[torch.device] = None) -> int:
    """Global family master over every rank's members: lowest deviation,
    ties to the lowest request id."""
    world = dist.get_world_size(group)
    device = device or (torch.device("cuda", torch.cuda.current_device())
                        if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    n_local = torch.tensor([len(local_scores)], dtype=torch.int64, device=device)
    counts = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(counts, n_local, group=group)
    width = int(max(c.item() for c in counts))
    if width == 0:
        raise ValueError("cannot elect a master from an empty group")
    buf = torch.full((width, 2), float("inf"), dtype=torch.float64, device=device)
    for i, (rid, score) in enumerate(sorted(local_scores.items())):
        buf[i, 0] = float(score)
        buf[i, 1] = float(rid)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    pairs = [(float(s), int(r)) for part in parts for s, r in part.tolist() if s != float("inf")]
    return min(pairs)[1]


# ---------------------------------------------------------------------------
# family master exchange (SURVEY §8e collective 3)


def family_master_transfers(member_rank: Dict[int, int], master_id: int) -> Tuple[int, List[int]]:
    """(source rank, destination ranks) of one family's master cache: the
    rank holding the elected master sends it to every other rank holding at
    least one mirror of the family."""
    src = member_rank[master_id]
    dsts = sorted({r for rid, r in member_rank.items() if rid != master_id and r != src})
    return src, dsts


def exchange_family_master(master_planes, like: Optional[Tuple[torch.Tensor, torch.Tensor]],
                           src: int, dsts: Sequence[int], rank: int, group=None):
    """Move the family master's dense (L, T, H, D) K and V planes from
    ``src`` to ``dsts`` (NCCL send/recv between GPUs; gloo stages CUDA
    tensors through host memory).  ``master_planes`` is (k, v) on ``src``;
    destinations allocate the receive buffers shaped like ``like`` (one of
    their local mirrors: a family's members share every dimension).  Returns
    the (k, v) planes on ``src`` and every destination, None elsewhere.
    Bytes received per destination: 2 * L*T*H*D * elt."""
    if rank != src and rank not in dsts:
        return None
    staged = dist.get_backend(group) == "gloo"
    ops, fix = [], []
    if rank == src:
        k, v = master_planes
        k, v = k.contiguous(), v.contiguous()
        send = (k.cpu(), v.cpu()) if staged and k.is_cuda else (k, v)
        for d in dsts:
            for t in send:
                ops.append(dist.P2POp(dist.isend, t, d, group=group))
        out = (k, v)
    else:
        ref_k, ref_v = like
        k = torch.empty(ref_k.shape, dtype=ref_k.dtype, device=ref_k.device)
        v = torch.empty(ref_v.shape, dtype=ref_v.dtype, device=ref_v.device)
        for t in (k, v):
            if staged and t.is_cuda:
                buf = torch.empty(t.shape, dtype=t.dtype)
                ops.append(dist.P2POp(dist.irecv, buf, src, group=group))
                fix.append((buf, t))
            else:
                ops.append(dist.P2POp(dist.irecv, t, src, group=group))
        out = (k, v)
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        for buf, t in fix:
            t.copy_(buf)
    return out


def encode_family_sharded(local_kv: Dict[int, object], local_hints: Dict[int, object],
                          local_scores: Dict[int, float], member_rank: Dict[int, int],
                          encode: Callable, make_kv: Callable, group=None,
                          device: Optional[torch.device] = None):
    """One family spread over ranks, encoded as DiffStore.encode_family does
    in one process (diffstore.py:411-439): elect the master over every rank's
    deviation scores (collective.py:117-121), ship the master's dense cache
    to the ranks holding mirrors, and encode this rank's mirrors (ascending
    request id) against it.

    ``local_kv``: rid -> LayeredKv of this rank's members; ``member_rank``:
    rid -> rank for the whole family (known to every rank: the agent
    sharding is deterministic); ``encode(master_kv, mirrors, hints)`` is the
    batched encoder (``encode_batch`` on the GPU); ``make_kv(k, v,
    positions)`` wraps received planes.  Returns (master_id, {rid: diff})
    for this rank's mirrors."""
    rank = dist.get_rank(group)
    master_id = elect_master(local_scores, group=group, device=device)
    src, dsts = family_master_transfers(member_rank, master_id)
    mirrors = sorted(rid for rid in local_kv if rid != master_id)
    if rank == src:
        mkv = local_kv[master_id]
        exchange_family_master((mkv.k, mkv.v), None, src, dsts, rank, group)
    elif mirrors:
        like = local_kv[mirrors[0]]
        k, v = exchange_family_master(None, (like.k, like.v), src, dsts, rank, group)
        mkv = make_kv(k, v, like.positions)
    if not mirrors:
        return master_id, {}
    diffs = encode(mkv, [local_kv[r] for r in mirrors], [local_hints[r] for r in mirrors])
    return master_id, dict(zip(mirrors, diffs))
