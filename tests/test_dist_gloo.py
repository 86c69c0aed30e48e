"""World-size-2 gloo tests of the multi-GPU host logic on CPU: agent
sharding, the master-arena broadcast, master election, and that the union
of per-shard collector outputs equals the single-process output."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import roundkv_port as ref
from paper_2604_03143_b200 import rounds
from paper_2604_03143_b200.dist import broadcast_arena, elect_master, shard_range
from paper_2604_03143_b200.paged_pool import choose_slots

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _Arena:
    def __init__(self, k, v):
        self.k, self.v = k, v


def _oracle_shard(spec, agents, mk, mv):
    """Oracle collector for ``agents`` with each agent's slots from the
    reference allocator replayed on this shard's pool."""
    T = spec.tokens_per_agent
    free = np.ones(len(agents) * T, bool)
    pk = np.zeros((spec.num_layers, free.size, spec.num_heads, spec.head_dim), np.float32)
    pv = np.zeros_like(pk)
    out = {}
    for a in agents:
        slots = choose_slots(free, T, 32)
        free[slots] = False
        jobs = []
        for cj in rounds.agent_jobs(spec, a, slots):
            r0 = cj.segment * spec.seg_len
            jobs.append(ref.CollectJob(0, mk[:, r0:r0 + spec.seg_len], mv[:, r0:r0 + spec.seg_len],
                                       np.arange(spec.seg_len), cj.delta))
        ref.collect_into_pool(jobs, [slots], pk, pv, 10000.0)
        out[a] = (pk[:, slots].copy(), pv[:, slots].copy())
    return out


def _worker(rank, port, spec, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        mk, mv = rounds.master_planes_host(spec)
        if rank == 0:
            k, v = torch.from_numpy(mk.copy()), torch.from_numpy(mv.copy())
        else:
            k, v = torch.zeros(mk.shape), torch.zeros(mv.shape)
        arena = _Arena(k, v)
        nbytes = broadcast_arena(arena, 0)
        assert nbytes == 2 * mk.nbytes
        assert torch.equal(arena.k, torch.from_numpy(mk)) and torch.equal(arena.v, torch.from_numpy(mv))
        agents = shard_range(spec.num_agents, rank, WORLD)
        shard = _oracle_shard(spec, list(agents), arena.k.numpy(), arena.v.numpy())
        # local deviation scores -> every rank elects the same master
        scores = {a: float((a * 7919) % 13) / 4.0 for a in agents}
        master = elect_master(scores)
        results[rank] = (list(agents), {a: (kk.sum(), vv.sum()) for a, (kk, vv) in shard.items()},
                         master)
    finally:
        dist.destroy_process_group()


def test_sharded_round_equals_single_process():
    spec = rounds.RoundSpec("gloo", 2, 2, 8, "f32", 5, 3, 7, 4)
    port = _free_port()
    with mp.Manager() as manager:
        results = manager.dict()
        mp.spawn(_worker, args=(port, spec, results), nprocs=WORLD, join=True)
        results = dict(results)
    shards = [results[r][0] for r in range(WORLD)]
    assert sorted(a for s in shards for a in s) == list(range(spec.num_agents))
    assert not set(shards[0]) & set(shards[1])
    mk, mv = rounds.master_planes_host(spec)
    whole = _oracle_shard(spec, list(range(spec.num_agents)), mk, mv)
    for r in range(WORLD):
        for a, (ks, vs) in results[r][1].items():
            assert ks == whole[a][0].sum() and vs == whole[a][1].sum()
    scores = {a: float((a * 7919) % 13) / 4.0 for a in range(spec.num_agents)}
    want = ref.select_master(scores)
    assert results[0][2] == results[1][2] == want


def test_shard_ranges_cover_agents():
    for n in (1, 5, 50, 1000):
        for world in (1, 2, 4, 8):
            got = [a for r in range(world) for a in shard_range(n, r, world)]
            assert got == list(range(n))
