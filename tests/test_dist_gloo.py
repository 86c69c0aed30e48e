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


class _LayeredArena(_Arena):
    @property
    def num_layers(self):
        return self.k.shape[0]


def _exchange_worker(rank, world, port, spec, results):
    from paper_2604_03143_b200.dist import exchange_sessions, session_transfers
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mk, mv = rounds.master_planes_host(spec)
        owners = rounds.session_owners(spec, world)
        needs = rounds.session_needs(spec, world)
        k, v = torch.zeros(mk.shape), torch.zeros(mv.shape)
        for s in range(spec.sessions):          # a rank starts with the masters it owns
            if owners[s] == rank:
                r0, r1 = spec.session_rows(s)
                k[:, r0:r1] = torch.from_numpy(mk[:, r0:r1])
                v[:, r0:r1] = torch.from_numpy(mv[:, r0:r1])
        arena = _LayeredArena(k, v)
        transfers = session_transfers(owners, needs)
        rows = [spec.session_rows(s) for s in range(spec.sessions)]
        dist.barrier()
        # two layer chunks, as exchange_collect posts them
        for chunk in ((0, 1), (1, spec.num_layers)):
            for r in exchange_sessions(arena, rows, transfers, rank, chunk):
                r.wait()
        have = []
        for s in range(spec.sessions):
            r0, r1 = spec.session_rows(s)
            have.append(bool(torch.equal(k[:, r0:r1], torch.from_numpy(mk[:, r0:r1]))
                             and torch.equal(v[:, r0:r1], torch.from_numpy(mv[:, r0:r1]))))
        agents = list(rounds.shard(spec.num_agents, rank, world))
        shard = _oracle_shard(spec, agents, k.numpy(), v.numpy())
        results[rank] = (agents, have, transfers,
                         {a: (kk.sum(), vv.sum()) for a, (kk, vv) in shard.items()})
    finally:
        dist.destroy_process_group()


def test_session_exchange_strong_shards():
    """Multi-session round sharded by agent (strong scaling): every rank ends
    with exactly the sessions its shard reads, and the shards' collector
    outputs equal a single-process round."""
    world = 3
    spec = rounds.RoundSpec("gloo-sessions", 2, 2, 8, "f32", 11, 2, 5, 3, sessions=4, strong=True)
    port = _free_port()
    with mp.Manager() as manager:
        results = manager.dict()
        mp.spawn(_exchange_worker, args=(world, port, spec, results), nprocs=world, join=True)
        results = dict(results)
    needs = rounds.session_needs(spec, world)
    owners = rounds.session_owners(spec, world)
    assert results[0][2], "the test round must exercise at least one transfer"
    for r in range(world):
        agents, have, _, sums = results[r]
        assert agents == list(rounds.shard(spec.num_agents, r, world))
        for s in range(spec.sessions):
            if s in needs[r] or owners[s] == r:
                assert have[s], (r, s)
            else:
                assert not have[s], (r, s)      # nothing beyond what the shard reads
    mk, mv = rounds.master_planes_host(spec)
    whole = _oracle_shard(spec, list(range(spec.num_agents)), mk, mv)
    for r in range(world):
        for a, (ks, vs) in results[r][3].items():
            assert ks == whole[a][0].sum() and vs == whole[a][1].sum()


def test_session_owners_and_bytes():
    spec = rounds.CONFIGS["c3"]
    for world in (1, 2, 4, 8):
        owners = rounds.session_owners(spec, world)
        needs = rounds.session_needs(spec, world)
        for s, o in enumerate(owners):
            assert s in needs[o]
        # contiguous shards: a rank reads at most one session beyond its share
        assert max(len(n) for n in needs) <= -(-spec.sessions // world) + 1
        total = sum(spec.collector_bytes_for(rounds.shard(spec.num_agents, r, world))
                    for r in range(world))
        assert total >= spec.collector_bytes()


def test_peer_unit_sources_follow_segment_owners():
    """Peer-read rounds: every collect unit is read from the rank owning its
    segment (host planning only; the IPC mapping and the multi-source K1 are
    exercised by tests/test_gpu_dist.py)."""
    from paper_2604_03143_b200.collector import _build_units, unit_sources
    from paper_2604_03143_b200.peer import contiguous_owners
    assert contiguous_owners(16, 8).tolist() == [0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7]
    assert contiguous_owners(5, 2).tolist() == [0, 0, 0, 1, 1]
    seg_len = np.array([40, 0, 17, 256, 3], np.int64)
    seg_row0 = np.concatenate([[0], np.cumsum(seg_len)[:-1]])
    owners = np.array([1, 0, 0, 3, 2])
    jobs_seg = np.sort(np.random.default_rng(0).choice([0, 2, 3, 4], 30))
    units, _ = _build_units(seg_row0, seg_len, jobs_seg, 3, 8, 64)
    src = unit_sources(units["row0"], seg_row0, seg_len, owners)
    seg_of = np.searchsorted(np.cumsum(seg_len), units["row0"], side="right")
    assert src.dtype == np.uint8
    assert src.tolist() == owners[seg_of].tolist()
    with pytest.raises(ValueError):
        unit_sources(np.array([int(seg_len.sum())]), seg_row0, seg_len, owners)


class _Kv:
    """A member cache as the exchange sees it: torch planes + positions."""

    def __init__(self, k, v, positions):
        self.k, self.v, self.positions = k, v, positions


def _family_members(n, seed=11, L=2, T=75, H=2, D=8, bs=16):
    """Master-like base cache; member i re-draws its own blocks (a family
    whose members differ from each other in a few blocks each)."""
    rng = np.random.default_rng(seed)
    base_k = rng.standard_normal((L, T, H, D)).astype(np.float32)
    base_v = rng.standard_normal((L, T, H, D)).astype(np.float32)
    nb = -(-T // bs)
    kvs, changed = {}, {}
    for rid in range(n):
        k, v = base_k.copy(), base_v.copy()
        blocks = sorted(rng.choice(nb, 2, replace=False).tolist())
        for b in blocks:
            k[:, b * bs:(b + 1) * bs] = rng.standard_normal(k[:, b * bs:(b + 1) * bs].shape)
            v[:, b * bs:(b + 1) * bs] = rng.standard_normal(v[:, b * bs:(b + 1) * bs].shape)
        kvs[rid] = (k, v)
        changed[rid] = blocks
    scores = {rid: float(rng.integers(0, 5)) for rid in range(n)}   # ties -> lowest id
    return kvs, changed, scores, bs


def _hints_vs(master_blocks, own_blocks, T, bs):
    blocks = sorted(set(master_blocks) | set(own_blocks))
    return np.concatenate([np.arange(b * bs, min(T, b * bs + bs)) for b in blocks])


def _family_worker(rank, world, port, n, member_rank, results):
    from paper_2604_03143_b200.dist import encode_family_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kvs, changed, scores, bs = _family_members(n)
        T = kvs[0][0].shape[1]
        master_id = ref.select_master(scores)       # hints need it: every member vs the master
        mine = [rid for rid in range(n) if member_rank[rid] == rank]
        local_kv = {rid: _Kv(torch.from_numpy(kvs[rid][0]), torch.from_numpy(kvs[rid][1]),
                             np.arange(T)) for rid in mine}
        local_hints = {rid: _hints_vs(changed[master_id], changed[rid], T, bs) for rid in mine}

        def encode(m, mirrors, hints):
            return [ref.encode_diff(m.k.numpy(), m.v.numpy(), x.k.numpy(), x.v.numpy(), h, bs)
                    for x, h in zip(mirrors, hints)]

        got_master, diffs = encode_family_sharded(
            local_kv, local_hints, {rid: scores[rid] for rid in mine}, member_rank, encode,
            lambda k, v, pos: _Kv(k, v, pos))
        results[rank] = (got_master, {rid: [(d.indices.tolist(), d.k_blocks.tobytes(),
                                             d.v_blocks.tobytes()) for d in layers]
                                      for rid, layers in diffs.items()})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,member_rank", [
    (2, {0: 0, 1: 0, 2: 1, 3: 1, 4: 1}),           # contiguous shards
    (3, {0: 2, 1: 0, 2: 1, 3: 2, 4: 0, 5: 1}),     # master off rank 0, scattered members
])
def test_family_master_exchange_equals_single_process_encode(world, member_rank):
    """A family spread over ranks (SURVEY §8e collective 3): every rank
    elects the same master, receives its dense cache from the rank holding
    it, and encodes its own mirrors against it; the union of the per-rank
    diffs equals a single-process encode_family (diffstore.py:411-439) bit
    for bit."""
    n = len(member_rank)
    port = _free_port()
    with mp.Manager() as manager:
        results = manager.dict()
        mp.spawn(_family_worker, args=(world, port, n, member_rank, results), nprocs=world,
                 join=True)
        results = dict(results)
    kvs, changed, scores, bs = _family_members(n)
    T = kvs[0][0].shape[1]
    master_id = ref.select_master(scores)
    assert {results[r][0] for r in range(world)} == {master_id}
    union = {}
    for r in range(world):
        assert not set(union) & set(results[r][1])
        union.update(results[r][1])
    assert sorted(union) == [rid for rid in range(n) if rid != master_id]
    mk, mv = kvs[master_id]
    for rid, got in union.items():
        want = ref.encode_diff(mk, mv, kvs[rid][0], kvs[rid][1],
                               _hints_vs(changed[master_id], changed[rid], T, bs), bs)
        assert got == [(d.indices.tolist(), d.k_blocks.tobytes(), d.v_blocks.tobytes())
                       for d in want]
    src = member_rank[master_id]
    from paper_2604_03143_b200.dist import family_master_transfers
    s, dsts = family_master_transfers(member_rank, master_id)
    assert s == src and src not in dsts
