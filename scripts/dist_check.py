"""Multi-rank collector check (launched by tests/test_gpu_dist.py via torchrun).

Each rank owns a contiguous agent shard; rank 0 alone holds the master
blocks and broadcasts them in layer chunks while every rank collects its
shard (dist.broadcast_collect).  Every rank then rebuilds its shard with a
single-process collect from the true masters and requires bit equality.
Backend: nccl on multi-GPU boxes, gloo when ranks share one GPU.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_03143_b200 as tk  # noqa: E402
from paper_2604_03143_b200 import rounds  # noqa: E402
from paper_2604_03143_b200.dist import (broadcast_collect, elect_master, exchange_collect,  # noqa: E402
                                        session_transfers, shard_range)


def main():
    backend = os.environ.get("TDKV_DIST_BACKEND", "gloo")
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group(backend)
    spec = rounds.CONFIGS["c2"].scaled(num_layers=5, num_agents=9, num_segments=3, hist_len=11)
    mk, mv = rounds.master_planes_host(spec)
    dt = spec.torch_dtype
    k = torch.from_numpy(mk).to(dev).to(dt)
    v = torch.from_numpy(mv).to(dev).to(dt)
    truth = rounds.make_arena(spec, k.clone(), v.clone())
    if rank != 0:
        k.zero_()
        v.zero_()
    arena = rounds.make_arena(spec, k, v)
    agents = shard_range(spec.num_agents, rank, world)
    T = spec.tokens_per_agent
    pool = tk.PagedPool(len(agents) * T + 8, spec.num_layers, spec.num_heads, spec.head_dim,
                        dtype=dt, device=dev)
    maps = [pool.allocate(T, a) for a in agents]
    jobs = [j for a, m in zip(agents, maps) for j in rounds.agent_jobs(spec, a, m.slots)]
    col = tk.KVCollector(arena, pool)
    plan = col.plan(jobs)
    broadcast_collect(col, plan, 0, chunks=3)
    torch.cuda.synchronize(dev)
    assert torch.equal(arena.k, truth.k) and torch.equal(arena.v, truth.v), "broadcast"
    ref_pool = tk.PagedPool(len(agents) * T + 8, spec.num_layers, spec.num_heads, spec.head_dim,
                            dtype=dt, device=dev)
    for a in agents:
        ref_pool.allocate(T, a)
    rc = tk.KVCollector(truth, ref_pool)
    rc.collect(rc.plan(jobs))
    torch.cuda.synchronize(dev)
    assert torch.equal(pool.k, ref_pool.k) and torch.equal(pool.v, ref_pool.v), "collect"
    dump = os.environ.get("TDKV_DIST_DUMP")
    if dump:
        # this rank's pool rows of every job, for the test to check against
        # the CPU oracle (tests/test_gpu_dist.py)
        rows = np.concatenate([np.asarray(j.dst_rows, np.int64) for j in jobs])
        sel = torch.from_numpy(rows).to(dev)
        np.savez(os.path.join(dump, f"rank{rank}.npz"), agents=np.asarray(list(agents)),
                 slots=np.stack([m.slots for m in maps]),
                 k=pool.k[:, sel].float().cpu().numpy(), v=pool.v[:, sel].float().cpu().numpy())
    scores = {a: float((a * 7919) % 13) / 4.0 for a in agents}
    master = elect_master(scores, device=dev if backend == "nccl" else torch.device("cpu"))
    want = min(((float((a * 7919) % 13) / 4.0, a) for a in range(spec.num_agents)))[1]
    assert master == want, (master, want)
    check_sessions(rank, world, dev)
    check_peer(rank, world, dev)
    check_family(rank, world, dev)
    dist.barrier()
    if rank == 0:
        print(f"dist_check ok: world={world} backend={backend}")
    dist.destroy_process_group()


def check_sessions(rank, world, dev):
    """Strong-scaling multi-session round: each rank starts with only the
    sessions it owns; exchange_collect moves the others point-to-point, layer
    chunk by layer chunk, and collects two pool sub-batches."""
    spec = rounds.CONFIGS["c3"].scaled(num_layers=3, num_agents=11, num_segments=2, seg_len=20,
                                       hist_len=5, sessions=4)
    mk, mv = rounds.master_planes_host(spec)
    dt = spec.torch_dtype
    k = torch.from_numpy(mk).to(dev).to(dt)
    v = torch.from_numpy(mv).to(dev).to(dt)
    truth = rounds.make_arena(spec, k.clone(), v.clone())
    owners = rounds.session_owners(spec, world)
    needs = rounds.session_needs(spec, world)
    for s in range(spec.sessions):
        if owners[s] != rank:
            r0, r1 = spec.session_rows(s)
            k[:, r0:r1] = 0
            v[:, r0:r1] = 0
    arena = rounds.make_arena(spec, k, v)
    agents = list(rounds.shard(spec.num_agents, rank, world))
    T = spec.tokens_per_agent
    sb = max(1, (len(agents) + 1) // 2)
    batches = [agents[i:i + sb] for i in range(0, len(agents), sb)]
    pools, plans = [], []
    for b in batches:
        pool = tk.PagedPool(len(b) * T + 8, spec.num_layers, spec.num_heads, spec.head_dim,
                            dtype=dt, device=dev)
        maps = [pool.allocate(T, a) for a in b]
        pools.append(pool)
        plans.append([j for a, m in zip(b, maps) for j in rounds.agent_jobs(spec, a, m.slots)])
    transfers = session_transfers(owners, needs)
    rows = [spec.session_rows(s) for s in range(spec.sessions)]
    for pool, jobs in zip(pools, plans):
        col = tk.KVCollector(arena, pool)
        exchange_collect(col, [col.plan(jobs)], rows, transfers, rank, chunks=2)
    torch.cuda.synchronize(dev)
    for s in needs[rank]:
        r0, r1 = spec.session_rows(s)
        assert torch.equal(arena.k[:, r0:r1], truth.k[:, r0:r1]), ("session", s)
    for pool, jobs in zip(pools, plans):
        ref_pool = tk.PagedPool(pool.capacity, spec.num_layers, spec.num_heads, spec.head_dim,
                                dtype=dt, device=dev)
        rc = tk.KVCollector(truth, ref_pool)
        rc.collect(rc.plan(jobs))
        torch.cuda.synchronize(dev)
        assert torch.equal(pool.k, ref_pool.k) and torch.equal(pool.v, ref_pool.v), "sessions"


def check_peer(rank, world, dev):
    """Peer-read rounds (peer.PeerRound): each rank holds only the segments it
    produced; K1 stages every other segment's tiles straight from the owner's
    arena (CUDA IPC mapping; NVLink between GPUs, the same HBM when the ranks
    share one GPU).  Two rounds with fresh masters check the ready/done
    protocol; every rank's pool must equal a single-process collect."""
    from paper_2604_03143_b200.peer import PeerRound, contiguous_owners
    spec = rounds.CONFIGS["c2"].scaled(num_layers=4, num_agents=7, num_segments=5, hist_len=9)
    dt = spec.torch_dtype
    owners = contiguous_owners(spec.num_segments, world)
    mk, mv = rounds.master_planes_host(spec)
    k = torch.zeros(mk.shape, dtype=dt, device=dev)
    v = torch.zeros(mv.shape, dtype=dt, device=dev)
    arena = rounds.make_arena(spec, k, v)
    agents = shard_range(spec.num_agents, rank, world)
    T = spec.tokens_per_agent
    pool = tk.PagedPool(len(agents) * T + 8, spec.num_layers, spec.num_heads, spec.head_dim,
                        dtype=dt, device=dev)
    maps = [pool.allocate(T, a) for a in agents]
    jobs = [j for a, m in zip(agents, maps) for j in rounds.agent_jobs(spec, a, m.slots)]
    col = tk.KVCollector(arena, pool)
    plan = col.plan(jobs)
    peer = PeerRound(col, owners)
    for rnd in range(2):
        full_k = torch.from_numpy(mk).to(dev).to(dt) * (1 + rnd)
        full_v = torch.from_numpy(mv).to(dev).to(dt) - rnd
        for s in range(spec.num_segments):        # this rank "produces" its segments
            if owners[s] == rank:
                r0 = int(arena.seg_row0[s])
                r1 = r0 + int(arena.seg_len[s])
                k[:, r0:r1] = full_k[:, r0:r1]
                v[:, r0:r1] = full_v[:, r0:r1]
        peer.round(plan)
        torch.cuda.synchronize(dev)
        truth = rounds.make_arena(spec, full_k, full_v)
        ref_pool = tk.PagedPool(pool.capacity, spec.num_layers, spec.num_heads, spec.head_dim,
                                dtype=dt, device=dev)
        for a in agents:
            ref_pool.allocate(T, a)
        rc = tk.KVCollector(truth, ref_pool)
        rc.collect(rc.plan(jobs))
        torch.cuda.synchronize(dev)
        assert torch.equal(pool.k, ref_pool.k) and torch.equal(pool.v, ref_pool.v), ("peer", rnd)
    want = sum(int(arena.seg_len[s]) for s in range(spec.num_segments) if owners[s] != rank)
    row = spec.num_heads * spec.head_dim * k.element_size()
    assert peer.peer_bytes(plan) == 2 * spec.num_layers * row * want
    dist.barrier()


def check_family(rank, world, dev):
    """Family master exchange (SURVEY §8e collective 3): 7 bf16 members of
    one family spread over the ranks; the elected master's dense cache goes
    from its rank to the ranks holding mirrors, each rank encodes its mirrors
    with encode_batch (K2), and the union equals a single-process encode of
    the whole family bit for bit (indices and payload)."""
    from paper_2604_03143_b200.dist import encode_family_sharded
    L, T, H, D, bs, n = 3, 300, 4, 128, 32, 7
    g = torch.Generator(device="cpu").manual_seed(5)
    base_k = torch.randn((L, T, H, D), generator=g).to(torch.bfloat16)
    base_v = torch.randn((L, T, H, D), generator=g).to(torch.bfloat16)
    nb = -(-T // bs)
    kvs, hints = {}, {}
    for rid in range(n):
        k, v = base_k.clone(), base_v.clone()
        b = (3 * rid) % nb
        k[:, b * bs:(b + 1) * bs] += 1.0
        v[:, b * bs:(b + 1) * bs] -= 1.0
        kvs[rid] = tk.LayeredKv(k.to(dev), v.to(dev), np.arange(T))
        hints[rid] = np.arange(T)               # every block hinted
    scores = {rid: float((rid * 5 + 3) % n) for rid in range(n)}
    member_rank = {rid: (rid * world) // n for rid in range(n)}
    mine = [rid for rid in range(n) if member_rank[rid] == rank]
    blocks = tk.CacheBlockConfig(bs)
    master_id, diffs = encode_family_sharded(
        {r: kvs[r] for r in mine}, {r: hints[r] for r in mine}, {r: scores[r] for r in mine},
        member_rank, lambda m, mirs, hs: tk.encode_batch(m, mirs, hs, blocks),
        lambda k, v, pos: tk.LayeredKv(k, v, pos),
        device=dev if dist.get_backend() == "nccl" else torch.device("cpu"))
    assert master_id == min((s, r) for r, s in scores.items())[1]
    mirrors = [r for r in range(n) if r != master_id]
    whole = tk.encode_batch(kvs[master_id], [kvs[r] for r in mirrors], [hints[r] for r in mirrors],
                            blocks)
    want = dict(zip(mirrors, whole))
    assert sorted(diffs) == [r for r in mine if r != master_id]
    for rid, d in diffs.items():
        w = want[rid]
        assert [x.indices.tolist() for x in d.layers] == [x.indices.tolist() for x in w.layers]
        for a, b in zip(d.layers, w.layers):
            assert torch.equal(a.k_blocks, b.k_blocks) and torch.equal(a.v_blocks, b.v_blocks)
    dist.barrier()


if __name__ == "__main__":
    main()
