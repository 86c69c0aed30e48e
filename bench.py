#!/usr/bin/env python
"""Benchmark: collected-KV GB/s and agents/s per All-Gather round, plus the
diff codec's GB/s, on B200 (BASELINE.json metric).

A step is one All-Gather round of the KV Collector over the configured
synthetic round (default C3, north_star's target: Qwen2.5-14B-shaped bf16 KV
(48 layers, 8 KV heads, d=128), 250 agents in 10 sessions of 25, 25 shared
20-token blocks per session; C2 = Qwen2.5-7B-shaped, 50 agents x 16 shared
256-token blocks, is ``--config c2``): [N>1: the masters' exchange -- NCCL
broadcast / per-session send-recv overlapped with K1 per layer chunk, or with
--exchange p2p no transfer at all: K1 reads every tile from its owner over
NVLink] + K0 (cos/sin rows) + K1 (rotate + scatter into every agent's paged
slots).  ``value`` = algorithmic bytes (M + N*M per GPU) of all
ranks / max-over-ranks device time.  Agents are sharded: weak scaling (each
GPU owns a config's worth of agents: C1, C2, C4) or strong scaling (the
config's agents split over the GPUs: C3's 250 agents in 10 sessions, C5's
1000 agents collected in pool sub-batches of 125).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--exchange p2p]
    python bench.py --impl reference ...   # CPU oracle port on the host cores

Sub-benchmarks on the same line: the diff codec (encode, fused and dense
restore, TDDF wire), the check-layer selection (K4), the tensor-core
recompute (K5) and the grouped-vs-serial recovery of BASELINE configs[0].
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tdkv", choices=["tdkv", "reference"])
    ap.add_argument("--config", default="c3",
                    help="c1..c5 (default c3: north_star's Qwen2.5-14B-shaped 250-agent round)")
    ap.add_argument("--agents", type=int, default=0, help="agents per GPU (default: config)")
    ap.add_argument("--no-codec", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--mirror-frac", type=float, default=0.1)
    ap.add_argument("--codec-mirrors", type=int, default=49, help="mirrors per codec family")
    ap.add_argument("--codec-sweep", action="store_true",
                    help="encode/decode sweep over changed-block fractions (C4)")
    ap.add_argument("--profile", action="store_true", help="few launches, no extras (for ncu)")
    ap.add_argument("--rope-style", default="interleaved", choices=["interleaved", "neox"],
                    help="rotary pairing of the collector (the reference's interleaved pairs, "
                         "or rotate-half)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="N>1 master exchange: NCCL broadcast / send-recv into each rank's "
                         "arena, overlapped with K1 per layer chunk (nccl), or K1 reading "
                         "every master tile from its owner's arena over NVLink (p2p: "
                         "peer.PeerRound, CUDA IPC mappings, no received copy)")
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                    help="strong: the config's agents are sharded over the GPUs (C3, C5); "
                         "weak: every GPU owns a config's worth of agents (auto: per config)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during a region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, index: int, period: float = 0.002):
        self.index = index
        self.period = period
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:   # noqa: BLE001 - clocks are reported as unavailable
            self._nvml = None

    def _run(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:   # noqa: BLE001
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self._nvml is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:   # noqa: BLE001
        return 6650.0, "fallback"


def ncu_traffic(kernel: str, workload: str):
    """DRAM bytes per launch of ``kernel`` from the committed ncu capture of
    THIS workload (profiles/ncu_traffic.json) and the capture it came from;
    (None, None) when no capture of this workload exists -- never another
    config's figure."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            entry = json.load(f).get(workload, {}).get(kernel)
    except Exception:   # noqa: BLE001
        entry = None
    if not entry:
        return None, None
    return entry["dram_bytes_per_launch"], f"{entry.get('round')} {entry.get('report')}"


# ---------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference)


def _cpu_collect_agents(spec, agents, mk, mv):
    """Oracle collector (oracle/roundkv_port.collect_into_pool) for ``agents``
    of the round, each into its own f32 pool; returns elapsed seconds."""
    from oracle import roundkv_port as ref
    from paper_2604_03143_b200 import rounds
    T = spec.tokens_per_agent
    t0 = time.perf_counter()
    for a in agents:
        pk = np.empty((spec.num_layers, T, spec.num_heads, spec.head_dim), np.float32)
        pv = np.empty_like(pk)
        slots = np.arange(T, dtype=np.int64)
        jobs = []
        for cj in rounds.agent_jobs(spec, a, slots):
            r0 = cj.segment * spec.seg_len
            jobs.append(ref.CollectJob(0, mk[:, r0:r0 + spec.seg_len], mv[:, r0:r0 + spec.seg_len],
                                       np.arange(spec.seg_len), cj.delta))
        ref.collect_into_pool(jobs, [slots], pk, pv, 10000.0)
    return time.perf_counter() - t0


_REF_STATE = {}


def _ref_worker(args):
    agent, = args
    st = _REF_STATE
    return _cpu_collect_agents(st["spec"], [agent], st["mk"], st["mv"])


def cpu_masters(spec):
    """f32 masters on the host: the bf16-rounded values, upcast (the reference
    is float32-only, roundkv/core.py:180-181)."""
    import torch
    from paper_2604_03143_b200 import rounds
    mk, mv = rounds.master_planes_host(spec)
    if spec.dtype == "bf16":
        mk = torch.from_numpy(mk).bfloat16().float().numpy()
        mv = torch.from_numpy(mv).bfloat16().float().numpy()
    return mk, mv


def cpu_baseline(spec, seconds: float):
    mk, mv = cpu_masters(spec)
    # agents in order; a round smaller than the time budget (C1) is repeated
    # whole (each repetition re-reads the masters: M + n*M per round)
    done, rounds_done, elapsed = 0, 0, 0.0
    while elapsed < seconds:
        elapsed += _cpu_collect_agents(spec, [done], mk, mv)
        done += 1
        if done == spec.num_agents:
            rounds_done += 1
            done = 0
    nbytes = rounds_done * spec.collector_bytes(spec.num_agents) + (
        spec.collector_bytes(done) if done else 0)
    agents = rounds_done * spec.num_agents + done
    gbs = nbytes / elapsed / 1e9
    what = (f"{rounds_done} whole rounds" + (f" + {done} agents" if done else "")
            if rounds_done else f"the first {done} agents")
    return {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "port",
            "agents_per_s": round(agents / elapsed, 4),
            "sample": f"oracle collector (numpy, 1 thread, f32-upcast inputs) on {what} of "
                      f"{spec.name}: {elapsed:.1f} s; bytes counted at the config dtype "
                      f"(M + n*M per round)"}


def run_reference(args):
    """--impl reference: the oracle port of the reference path on all host
    cores (agents are independent; one process per core)."""
    import multiprocessing as mp
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2604_03143_b200 import rounds
    spec = rounds.CONFIGS[args.config]
    if args.agents:
        spec = spec.scaled(num_agents=args.agents)
    cores = len(os.sched_getaffinity(0))
    procs = max(1, min(cores, 32, spec.num_agents))
    mk, mv = cpu_masters(spec)
    _REF_STATE.update(spec=spec, mk=mk, mv=mv)
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        def step(i):
            agents = [((i * procs + j) % spec.num_agents,) for j in range(procs)]
            t0 = time.perf_counter()
            pool.map(_ref_worker, agents, chunksize=1)
            return time.perf_counter() - t0
        for i in range(args.warmup):
            step(i)
        times = [step(args.warmup + i) for i in range(args.steps)]
    t = sum(times) / len(times)
    gbs = spec.collector_bytes(procs) / t / 1e9
    line = {
        "impl": "reference", "metric": "collected KV GB/s", "value": round(gbs, 4),
        "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if spec.strong else "weak",
        "vs_baseline": None, "dtype": spec.dtype, "data": "synthetic",
        "config": {"workload": spec.name, "agents_per_step": procs},
        "agents_per_s": round(procs / t, 3),
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": procs, "kind": "port",
                         "sample": f"{procs} agents of {spec.name} per step, one process per "
                                   f"agent (oracle/roundkv_port, f32-upcast inputs)"},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# tdkv


def run_tdkv(args):
    import torch
    import torch.distributed as dist

    import paper_2604_03143_b200 as tk
    from paper_2604_03143_b200 import rounds
    from paper_2604_03143_b200.dist import (broadcast_arena, broadcast_collect,
                                            exchange_collect, exchange_sessions,
                                            session_transfers)

    world, rank, local = dist_env()
    # one GPU per rank; --dist-backend gloo lets a single-GPU box exercise the
    # multi-rank flow (ranks then share the device)
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    spec = rounds.CONFIGS[args.config]
    if args.agents:
        spec = spec.scaled(num_agents=args.agents)
    strong = spec.strong if args.scaling == "auto" else args.scaling == "strong"
    dt = spec.torch_dtype
    L, H, D = spec.num_layers, spec.num_heads, spec.head_dim
    T = spec.tokens_per_agent
    # strong: the config's agents are sharded over the ranks (contiguous, so a
    # session spans as few ranks as possible); weak: every rank owns a full
    # config's worth of agents
    if strong:
        agents = list(rounds.shard(spec.num_agents, rank, world))
    else:
        agents = list(range(rank * spec.num_agents, (rank + 1) * spec.num_agents))
    n_local = len(agents)
    sb = min(n_local, spec.sub_batch) if spec.sub_batch else n_local
    batches = [agents[i:i + sb] for i in range(0, n_local, sb)]

    # masters: host-pinned copy (the e2e input) + device arena
    mk_h, mv_h = rounds.master_planes_host(spec)
    host_k = torch.from_numpy(mk_h).to(dt).pin_memory()
    host_v = torch.from_numpy(mv_h).to(dt).pin_memory()
    del mk_h, mv_h
    arena = rounds.make_arena(spec, host_k.to(dev), host_v.to(dev))
    # the pool holds one sub-batch of agents; sub-batch j reuses its slots
    pool = tk.PagedPool(sb * T, L, H, D, dtype=dt, device=dev, debug=False)
    maps = [pool.allocate(T, a) for a in batches[0]]

    collector = tk.KVCollector(arena, pool, rope_style=args.rope_style)
    plans = [collector.plan([j for a, m in zip(b, maps) for j in rounds.agent_jobs(spec, a, m.slots)])
             for b in batches]
    plan = plans[0]
    step_bytes = sum(spec.collector_bytes_for(b) for b in batches)
    assert sum(p.algorithmic_bytes() for p in plans) == step_bytes

    # the round's one exchange (N>1): a single-session round broadcasts its
    # masters from rank 0; a multi-session round sends each session only to
    # the ranks whose shard reads it (point-to-point, NCCL over NVLink)
    owners = rounds.session_owners(spec, world) if strong else [0] * spec.sessions
    needs = (rounds.session_needs(spec, world) if strong
             else [list(range(spec.sessions))] * world)
    transfers = session_transfers(owners, needs)
    use_broadcast = spec.sessions == 1 or not strong
    session_rows = [spec.session_rows(s) for s in range(spec.sessions)]
    if use_broadcast:
        recv_bytes = spec.master_bytes if rank != 0 else 0
    else:
        recv_bytes = sum(spec.session_master_bytes for s, _, d in transfers if d == rank)

    # p2p: every rank holds only the masters it produced (segments of its
    # sessions / its contiguous share) and K1 reads the rest from the owners
    peer = None
    if world > 1 and args.exchange == "p2p":
        from paper_2604_03143_b200.peer import PeerRound, contiguous_owners
        if use_broadcast:
            seg_owner = contiguous_owners(spec.total_segments, world)
        else:
            seg_owner = np.repeat(np.asarray(owners, np.int64), spec.num_segments)
        for g in np.flatnonzero(seg_owner != rank):
            r0 = int(arena.seg_row0[g])
            arena.k[:, r0:r0 + int(arena.seg_len[g])] = 0
            arena.v[:, r0:r0 + int(arena.seg_len[g])] = 0
        torch.cuda.synchronize(dev)
        peer = PeerRound(collector, seg_owner)
        recv_bytes = peer.peer_bytes(plans[0]) if plans else 0
        if len(plans) > 1:
            recv_bytes = sum(peer.peer_bytes(p) for p in plans)

    stream = torch.cuda.current_stream(dev)

    # a round whose working set (masters read + pool rows written) would stay
    # resident in the 126 MB L2 across steps (C1) rotates over R independent
    # copies of the round (own arena, pool and plan; R x working set > 2 x
    # L2): every step's inputs were evicted by the R - 1 rounds before it,
    # and steps run back to back like a serving loop
    l2_size = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 0) or 0)
    l2_size = l2_size or 126 * 2**20
    working_set = spec.master_bytes + step_bytes
    rotation = [(collector, plans)]
    if working_set < 2 * l2_size and world == 1 and peer is None:
        for _ in range(-(-2 * l2_size // working_set)):
            arena_r = rounds.make_arena(spec, arena.k.clone(), arena.v.clone())
            pool_r = tk.PagedPool(sb * T, L, H, D, dtype=dt, device=dev, debug=False)
            maps_r = [pool_r.allocate(T, a) for a in batches[0]]
            col_r = tk.KVCollector(arena_r, pool_r, rope_style=args.rope_style)
            rotation.append((col_r, [col_r.plan([j for a, m in zip(b, maps_r)
                                                 for j in rounds.agent_jobs(spec, a, m.slots)])
                                     for b in batches]))
    rot_i = [0]

    def round_step(events=None):
        if events is not None:
            events[0].record(stream)
        if len(rotation) > 1:
            col_r, plans_r = rotation[rot_i[0] % len(rotation)]
            rot_i[0] += 1
            for p in plans_r:
                col_r.collect(p)
        elif peer is not None:
            # device-side round barriers around the peer-read collect
            peer.ready()
            for p in plans:
                peer.collect(p)
            peer.done()
        elif world > 1 and use_broadcast:
            # masters broadcast from rank 0 in layer chunks, K1 per landed chunk
            broadcast_collect(collector, plans, 0, chunks=7)
        elif world > 1:
            exchange_collect(collector, plans, session_rows, transfers, rank, chunks=4)
        else:
            for p in plans:
                collector.collect(p)
        if events is not None:
            events[1].record(stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def reduce_over_ranks(x: float, op) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64,
                         device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max_over_ranks(x: float) -> float:
        return reduce_over_ranks(x, dist.ReduceOp.MAX if world > 1 else None)

    total_bytes = int(reduce_over_ranks(float(step_bytes), dist.ReduceOp.SUM if world > 1 else None))
    total_agents = int(reduce_over_ranks(float(n_local), dist.ReduceOp.SUM if world > 1 else None))

    # -- device-timed rounds ------------------------------------------------
    for _ in range(args.warmup * len(rotation)):
        round_step()
    barrier()
    # per-step events bracket K1 when a step has more than the round's kernels
    # (N>1: the exchange); otherwise at N=1 a step IS the round (K0 + K1, or
    # K1 alone with the fused table) and the step time is K1's, without the
    # per-step event records' host cost
    per_step = world > 1
    k1_events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                 for _ in range(args.steps)] if per_step else [None] * args.steps
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = tk.launch_count()
    sampler = ClockSampler(local)
    with sampler:
        barrier()
        start.record(stream)
        for i in range(args.steps):
            round_step(k1_events[i])
        stop.record(stream)
        barrier()
    launches = tk.launch_count() - launches0
    elapsed_ms = max_over_ranks(start.elapsed_time(stop))
    ms_step = elapsed_ms / args.steps
    k1_ms = (sum(a.elapsed_time(b) for a, b in k1_events) / args.steps if per_step
             else start.elapsed_time(stop) / args.steps)
    value = total_bytes / (ms_step * 1e-3) / 1e9
    agents_per_s = total_agents / (ms_step * 1e-3)

    # the same round timed cold and alone (rotating rounds only): a 2 x L2
    # buffer written before each round, CUDA events around the round
    cold = None
    if len(rotation) > 1:
        flush_buf = torch.empty(2 * l2_size, dtype=torch.uint8, device=dev)
        cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for i in range(args.steps + args.warmup):
            flush_buf.fill_(1)
            if i >= args.warmup:
                cev[i - args.warmup][0].record(stream)
            round_step()
            if i >= args.warmup:
                cev[i - args.warmup][1].record(stream)
        torch.cuda.synchronize(dev)
        c_ms = sum(a.elapsed_time(b) for a, b in cev) / args.steps
        del flush_buf
        cold = {"ms_per_round": round(c_ms, 5),
                "value": round(step_bytes / (c_ms * 1e-3) / 1e9, 1), "unit": "GB/s",
                "note": "each round alone after a 2 x L2 buffer write (dirty L2, idle GPU, "
                        "launch ramp and tail inside the events)"}

    # the exchange alone (N>1): NVLink receive roofline of the busiest rank
    exchange = None
    if peer is not None:
        busiest = int(max_over_ranks(float(recv_bytes)))
        exchange = {"kind": "peer-read fused into K1 (tdkv_collect_sources over CUDA IPC "
                            "mappings)",
                    "peer_bytes_max_rank": busiest,
                    "nvlink_read_gbs": round(busiest / (ms_step * 1e-3) / 1e9, 1),
                    "peak": 900.0, "unit": "GB/s",
                    "note": "no separate transfer: the master tiles are TMA-staged from the "
                            "owner's HBM inside K1; two one-element NCCL all-reduces per round "
                            "are the ready/done barriers"}
    elif world > 1 and not args.profile:
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        x0.record(stream)
        for _ in range(args.steps):
            if use_broadcast:
                broadcast_arena(arena, 0)
            else:
                for r in exchange_sessions(arena, session_rows, transfers, rank):
                    r.wait()
        x1.record(stream)
        barrier()
        x_ms = max_over_ranks(x0.elapsed_time(x1)) / args.steps
        busiest = int(max_over_ranks(float(recv_bytes)))
        nvlink_peak = 900.0          # NVLink 5, GB/s per direction per GPU (nominal)
        exchange = {"kind": "broadcast" if use_broadcast else "session p2p",
                    "recv_bytes_max_rank": busiest, "ms": round(x_ms, 4),
                    "achieved": round(busiest / (x_ms * 1e-3) / 1e9, 1) if x_ms > 0 else None,
                    "peak": nvlink_peak, "unit": "GB/s",
                    "frac": round(busiest / (x_ms * 1e-3) / 1e9 / nvlink_peak, 4)
                    if x_ms > 0 else None,
                    "backend": args.dist_backend}

    # the family master exchange (N>1, SURVEY §8e collective 3): every family
    # (a session) elects its master -- here the session's first agent -- and
    # the rank holding that agent's cache sends its dense K/V to every other
    # rank holding members of the family, which then encode their mirrors
    # against it (dist.encode_family_sharded)
    if world > 1 and not args.profile and len(batches) == 1:
        line_family = family_exchange_bench(spec, pool, maps, agents, rank, world, dev, stream,
                                            barrier, max_over_ranks, args)
    else:
        line_family = None

    peak, peak_kind = measured_peak_hbm()
    achieved = step_bytes / (k1_ms * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic("collect_kernel", spec.name)
    line = {
        "metric": "collected KV GB/s", "value": round(value, 2), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": spec.dtype, "data": "synthetic",
        "config": {"workload": spec.name, "agents_per_gpu": n_local,
                   "total_agents": total_agents, "sessions": spec.sessions,
                   "sub_batches_per_gpu": len(batches), "shared_blocks": spec.num_segments,
                   "block_len": spec.seg_len, "layers": L, "kv_heads": H, "head_dim": D,
                   "tokens_per_agent": T, "parallelism": f"agent-shard x{world}",
                   "rope_pairs": args.rope_style,
                   "exchange": (None if world == 1 else
                                "p2p" if peer is not None else "nccl"),
                   "l2": (f"inputs larger than L2: steps rotate over {len(rotation)} "
                          "independent copies of the round (arena, pool, plan), "
                          f"{len(rotation) * working_set / 2**20:.0f} MiB in all vs "
                          f"{l2_size / 2**20:.0f} MiB of L2, so no step's data is "
                          "L2-resident when it starts" if len(rotation) > 1
                          else "inputs larger than L2 (master arena "
                          f"{spec.master_bytes / 2**20:.0f} MiB read, "
                          f"{step_bytes / 1e9:.1f} GB moved per GPU per step)")},
        "agents_per_s": round(agents_per_s, 1),
        "roofline": {"bound": "hbm", "kernel": "collect_kernel (K1)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": traffic_src,
                     "peak_source": peak_kind,
                     "algorithmic_bytes_per_launch": step_bytes,
                     "k1_ms": round(k1_ms, 4)},
        "gpu_launches": launches,
        "clocks": sampler.summary(),
    }
    if cold is not None:
        cold["frac"] = round(cold["value"] / peak, 4)
        line["cold_round"] = cold
    if exchange is not None:
        line["exchange"] = exchange
    if line_family is not None:
        line["family_exchange"] = line_family

    # -- the same rounds replayed from a captured CUDA graph (N=1) -----------
    if world == 1 and len(plans) == 1 and not args.profile:
        graphs = [col_r.capture(plans_r[0]) for col_r, plans_r in rotation]
        for _ in range(args.warmup):
            for g in graphs:
                g.replay()
        torch.cuda.synchronize(dev)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for i in range(args.steps):
            graphs[i % len(graphs)].replay()
        g1.record(stream)
        torch.cuda.synchronize(dev)
        g_ms = g0.elapsed_time(g1) / args.steps
        graph = graphs[0]
        line["graph"] = {"value": round(step_bytes / (g_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                         "ms_per_step": round(g_ms, 4), "kernels_per_replay": graph.kernels,
                         "note": "KVCollector.capture(plan): the round (K0 + K1) as one CUDA "
                                 "graph, replayed; not counted in gpu_launches"}
        del graph, graphs

    # -- e2e: public API with host buffers ---------------------------------
    if len(batches) > 1 and not args.no_e2e:
        line["e2e_note"] = ("e2e measured for single-sub-batch shards only (this shard is "
                            f"collected in {len(batches)} pool sub-batches)")
    if not args.no_e2e and not args.profile and len(batches) == 1:
        status = torch.empty(1, dtype=dt, device="cpu").pin_memory()

        # host metadata of the round: each agent's prompt layout (segment
        # start rows); the agents' slot maps are pool state, resident on the
        # device since admission (SlotArena)
        slot_arena = tk.SlotArena(maps, dev)
        first_slot = int(maps[0].slots[spec.hist_len + 1])
        copy_stream = torch.cuda.Stream(dev)
        done = torch.cuda.Event()

        # the agents' prompt layouts (segment offsets): host metadata the
        # round starts from; planning turns them into the round's jobs
        layouts = rounds.agent_starts(spec, agents)

        def plan_round():
            segs, dst_off, job_delta = rounds.round_offsets(spec, agents, slot_arena.base,
                                                            starts=layouts)
            return collector.plan_offsets(segs, dst_off, job_delta, slot_arena)

        def e2e_step():
            # plan from host metadata (tiny uploads, issued first), then the
            # shared blocks arrive from pinned host memory in layer chunks on
            # a copy stream while K1 runs on the landed chunks; the host reads
            # one result element back per round
            p = plan_round()
            events = collector.stage_from_host(host_k, host_v, chunks=7, copy_stream=copy_stream)
            collector.collect_staged(p, events)
            status.copy_(pool.k[0, first_slot].view(-1)[:1], non_blocking=True)
            done.record(stream)
            done.synchronize()
            return p

        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            p = e2e_step()
        barrier()
        single_wall = max_over_ranks(time.perf_counter() - t0) / args.steps

        # steady state: round r+1's masters stream in (copy stream, second
        # arena) while round r is collected; every step still carries one
        # round's H2D and one synchronous result read
        pipe = tk.RoundPipeline(arena, pool, chunks=7)

        def pipe_step():
            p = plan_round()
            pipe.step(p, host_k, host_v)
            status.copy_(pool.k[0, first_slot].view(-1)[:1], non_blocking=True)
            done.record(stream)
            done.synchronize()
            return p

        pipe.prime(host_k, host_v)
        for _ in range(max(1, args.warmup)):
            pipe_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            p = pipe_step()
        barrier()                      # includes the last in-flight H2D
        wall = max_over_ranks(time.perf_counter() - t0) / args.steps
        e2e_gbs = total_bytes / wall / 1e9
        # breakdown: the H2D alone (copy-stream events) and the host planning alone
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(copy_stream)
        collector.stage_from_host(host_k, host_v, chunks=7, copy_stream=copy_stream)
        h1.record(copy_stream)
        torch.cuda.synchronize(dev)
        h2d_ms = h0.elapsed_time(h1)
        tp = time.perf_counter()
        plan_round()
        torch.cuda.synchronize(dev)
        plan_ms = (time.perf_counter() - tp) * 1e3
        # the PCIe ceiling of this box: one pinned 512 MiB host -> HBM copy
        probe_h = torch.ones(1 << 29, dtype=torch.uint8).pin_memory()   # pages touched
        probe_d = torch.empty(1 << 29, dtype=torch.uint8, device=dev)
        for _ in range(2):                                            # untimed warm-up
            probe_d.copy_(probe_h, non_blocking=True)
        torch.cuda.synchronize(dev)
        ceil_ms = []
        for _ in range(5):
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            probe_d.copy_(probe_h, non_blocking=True)
            c1.record(stream)
            torch.cuda.synchronize(dev)
            ceil_ms.append(c0.elapsed_time(c1))
        del probe_h, probe_d
        h2d_ceiling = (1 << 29) / (min(ceil_ms) * 1e-3) / 1e9
        master_bytes_step = 2 * host_k.numel() * host_k.element_size()
        line["e2e"] = {"value": round(e2e_gbs, 2), "unit": "GB/s",
                       "h2d_gbs": round(master_bytes_step / wall / 1e9, 2),
                       "h2d_ceiling_gbs": round(h2d_ceiling, 2),
                       "h2d_frac": round(master_bytes_step / wall / 1e9 / h2d_ceiling, 4),
                       "h2d_bytes_per_step": int(2 * host_k.numel() * host_k.element_size()
                                                 + p.h2d_bytes),
                       "d2h_bytes_per_step": int(status.numel() * status.element_size()),
                       "ms_per_step": round(wall * 1e3, 3),
                       "h2d_ms": round(h2d_ms, 3), "plan_ms": round(plan_ms, 3),
                       "single_round_ms": round(single_wall * 1e3, 3),
                       "agents_per_s": round(total_agents / wall, 1),
                       "path": "per step: KVCollector.plan_offsets (host layouts -> job "
                               "records against the device-resident slot maps; ~30 KB "
                               "uploaded) + RoundPipeline.step (the next round's pinned-host "
                               "masters stream in 7 layer chunks on a copy stream into the "
                               "second arena while K0+K1 collect this round) + synchronous "
                               "result read; single_round_ms = the same without cross-round "
                               "overlap"}

    # -- codec sub-benchmarks (rank-local) ----------------------------------
    if not args.no_codec and not args.profile:
        line["codec"] = codec_bench(tk, spec, pool, maps, dev, args, peak)
        line["selection"] = selection_bench(tk, spec, pool, maps, dev, args, peak)
        if world == 1:
            line["dropin"] = dropin_bench(tk, args)
        line["recompute"] = recompute_bench(dev, args)
        line["recovery"] = recovery_bench(dev, args)
        if args.codec_sweep:
            line["codec_sweep"] = codec_sweep(tk, spec, pool, maps, dev, args, peak)

    if not args.no_codec and not args.profile and rank == 0:
        line["host_planning"] = planning_bench()

    if not args.no_cpu and not args.profile and rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline(spec, args.cpu_seconds)

    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def family_exchange_bench(spec, pool, maps, agents, rank, world, dev, stream, barrier,
                          max_over_ranks, args):
    """Time the family master exchange of one round: per family (session
    under strong scaling, the whole round otherwise) the master agent's dense
    cache -- gathered from its pool slots on the owning rank -- goes
    point-to-point to every other rank holding family members.  NVLink
    receive roofline of the busiest rank."""
    import torch
    import torch.distributed as dist
    from paper_2604_03143_b200 import dist as tdist
    strong = spec.sessions > 1
    if strong:
        rank_of = {a: r for r in range(world) for a in rounds_shard(spec, r, world)}
    else:                         # weak: each rank owns a full config's agents
        rank_of = {a: r for r in range(world)
                   for a in range(r * spec.num_agents, (r + 1) * spec.num_agents)}
    fams = {}
    for a, r in rank_of.items():
        fams.setdefault(spec.session_of(a % spec.num_agents) if strong else 0, {})[a] = r
    local = {a: m for a, m in zip(agents, maps)}
    T = spec.tokens_per_agent
    L, H, D = spec.num_layers, spec.num_heads, spec.head_dim
    plan = []
    for f, members in sorted(fams.items()):
        master = min(members)               # elected: synthetic deviations rank by id
        src, dsts = tdist.family_master_transfers(members, master)
        if rank == src or rank in dsts:
            plan.append((master, src, dsts))
    recv = sum(spec.dense_bytes for _, src, _ in plan if src != rank)   # K+V per family
    shape = (L, T, H, D)

    def one_round():
        outs = []
        for master, src, dsts in plan:
            if rank == src:
                sl = local[master].device_slots(dev)
                planes = (pool.k[:, sl], pool.v[:, sl])       # gather (K3-equivalent copy)
                outs.append(tdist.exchange_family_master(planes, None, src, dsts, rank))
            else:
                like = (torch.empty(shape, dtype=pool.dtype, device=dev),) * 2
                outs.append(tdist.exchange_family_master(None, like, src, dsts, rank))
        return outs

    one_round()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        one_round()
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    busiest = int(max_over_ranks(float(recv)))
    return {"families": len(fams), "families_touching_this_rank": len(plan),
            "recv_bytes_max_rank": busiest, "ms": round(ms, 4),
            "achieved": round(busiest / (ms * 1e-3) / 1e9, 1) if ms > 0 else None,
            "peak": 900.0, "unit": "GB/s",
            "frac": round(busiest / (ms * 1e-3) / 1e9 / 900.0, 4) if ms > 0 else None,
            "backend": args.dist_backend,
            "note": "master = the family's lowest agent id; its dense K/V (gathered from "
                    "the pool) sent point-to-point to the ranks holding mirrors "
                    "(dist.exchange_family_master)"}


def planning_bench(spec_name: str = "c5", agents: int = 0):
    """Host planning of one round from the reference's objects (SURVEY §8f
    #4): the round's PromptLayouts (C5: 1000 agents, each a 512-token private
    history + 16 shared 256-token outputs) -> native prepare_request of every
    prompt (tdkv_prepare_batch: flatten, segment-index lookups, labels,
    structural sets) -> the collector's job arrays -> the collector's unit
    plan (plan_host_offsets).  Host wall clock, median of 5; the oracle's
    pure-Python prepare_request restatement is timed on 40 prompts."""
    from oracle import roundkv_port as ref
    from paper_2604_03143_b200 import prepare as pp, rounds
    from paper_2604_03143_b200.collector import pick_tile_rows, plan_host_offsets
    spec = rounds.CONFIGS[spec_name]
    if agents:
        spec = spec.scaled(num_agents=agents)
    n = spec.num_agents
    sep = 151643                     # Qwen2.5's <|endoftext|>
    layouts, index, eseg = rounds.round_layouts(spec, range(n), sep)
    T = spec.tokens_per_agent
    base = np.arange(n, dtype=np.int64) * T
    seg_row0 = np.arange(spec.total_segments, dtype=np.int64) * spec.seg_len
    seg_len = np.full(spec.total_segments, spec.seg_len, np.int64)
    tile = pick_tile_rows(spec.row_bytes)

    class _M:
        separator_token = sep

    def native():
        t0 = time.perf_counter()
        preps = pp.prepare_requests(layouts, _M, index)
        t1 = time.perf_counter()
        batch = pp.prepare_batch(layouts, sep, index)
        segs, dst, delta = pp.plan_offsets_from_prepared(batch, eseg, base)
        t2 = time.perf_counter()
        plan_host_offsets(seg_row0, seg_len, segs, dst, delta, spec.num_layers, tile)
        t3 = time.perf_counter()
        return preps, (t1 - t0, t2 - t1, t3 - t2)

    native()
    runs = [native()[1] for _ in range(5)]
    med = [statistics.median(r[i] for r in runs) for i in range(3)]
    port_index = ref.SegmentIndexPort(1 << 62)
    for e in index.entries():
        port_index.insert(e)
    k = min(40, n)
    t0 = time.perf_counter()
    for lay in layouts[:k]:
        ref.prepare_request_port([(s.kind.value, s.tokens, s.digest) for s in lay.segments],
                                 sep, port_index.lookup)
    port_s = (time.perf_counter() - t0) / k
    total = med[1] + med[2]
    return {"workload": spec.name, "agents": n, "tokens_per_agent": T,
            "prepare_requests_ms": round(med[0] * 1e3, 3),
            "prepare_and_offsets_ms": round(med[1] * 1e3, 3),
            "unit_plan_ms": round(med[2] * 1e3, 3),
            "round_planning_ms": round(total * 1e3, 3),
            "agents_per_s": round(n / total, 1),
            "oracle_prepare_ms_per_agent": round(port_s * 1e3, 4),
            "oracle_prepare_round_ms_extrapolated": round(port_s * n * 1e3, 1),
            "note": "host wall clock, median of 5: prepare_requests = the drop-in "
                    "PreparedRequest objects of every prompt (one tdkv_prepare_batch "
                    "call); prepare_and_offsets = the native batch + the collector's job "
                    "arrays (segment, slot-arena offset, delta) from the hits; unit_plan = "
                    "plan_host_offsets; oracle = roundkv_port.prepare_request_port (the "
                    "reference's algorithm in Python) on 40 prompts, 1 core"}


def rounds_shard(spec, rank, world):
    from paper_2604_03143_b200 import rounds
    return rounds.shard(spec.num_agents, rank, world)


def dropin_bench(tk, args):
    """The reference contract end to end: ``skeleton_values`` +
    ``align_cached`` (pic.py:203-204, 208-235) on HOST numpy contexts -- the
    drop-in call a reference caller makes -- on BASELINE configs[0] (8 agents
    x 4 shared 256-token blocks, L=2, H=8, D=64, float32): masters and
    contexts go host -> HBM, K1 runs, the rows come back over PCIe into the
    numpy contexts.  Timed beside the oracle's collector on the same inputs
    (numpy, one host core)."""
    import torch
    from paper_2604_03143_b200 import rounds
    from oracle import roundkv_port as ref   # CPU timing leg only
    spec = rounds.CONFIGS["c1"]
    mk, mv = rounds.master_planes_host(spec)
    src = rounds.source_offsets(spec)
    L, H, D, n = spec.num_layers, spec.num_heads, spec.head_dim, spec.seg_len
    masters = [tk.LayeredKv(np.ascontiguousarray(mk[:, g * n:(g + 1) * n]),
                            np.ascontiguousarray(mv[:, g * n:(g + 1) * n]),
                            np.arange(src[g], src[g] + n)) for g in range(spec.total_segments)]

    class _Hit:
        def __init__(self, kv, target, delta):
            self.kv, self.target_idx, self.delta = kv, target, delta

    class _Member:
        def __init__(self, hits):
            self.hits = hits

    T = spec.tokens_per_agent
    members, jobs = [], []
    for a in range(spec.num_agents):
        starts = rounds.segment_starts(spec, a)
        hits = []
        for sgm in range(spec.num_segments):
            tgt = np.arange(starts[sgm], starts[sgm] + n, dtype=np.int64)
            delta = tgt - masters[sgm].positions
            hits.append(_Hit(masters[sgm], tgt, delta))
            jobs.append(ref.CollectJob(a, masters[sgm].k, masters[sgm].v, tgt, delta))
        members.append(_Member(hits))

    def fresh():
        return [(np.zeros((L, T, H, D), np.float32), np.zeros((L, T, H, D), np.float32))
                for _ in range(spec.num_agents)]

    def ours(ctx):
        tk.skeleton_values(members, ctx)
        tk.align_cached(members, ctx, 10000.0)

    for _ in range(3):
        ours(fresh())
    times = []
    for _ in range(max(5, min(args.steps, 20))):
        ctx = fresh()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ours(ctx)
        times.append(time.perf_counter() - t0)
    t_ours = float(np.median(times))
    # the same call into contexts whose pages are already touched (a caller
    # reusing its context buffers): what is left is PCIe + the device pass
    times = []
    ctx_warm = fresh()
    for c in ctx_warm:
        c[0].fill(1.0)
        c[1].fill(1.0)
    for _ in range(max(5, min(args.steps, 20))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ours(ctx_warm)
        times.append(time.perf_counter() - t0)
    t_warm = float(np.median(times))
    ctx_ref = fresh()
    t0 = time.perf_counter()
    ref.collect_into_contexts(jobs, ctx_ref, 10000.0)
    t_ref = time.perf_counter() - t0
    same_v = all(np.array_equal(a[1], b[1]) for a, b in zip(ctx, ctx_ref))
    err_k = max(float(np.abs(a[0] - b[0]).max()) for a, b in zip(ctx, ctx_ref))
    moved = spec.collector_bytes()
    return {"path": "skeleton_values + align_cached on host numpy contexts (the reference "
                    "contract): masters and rows over PCIe both ways",
            "config": spec.name, "ms_per_round": round(t_ours * 1e3, 3),
            "ms_per_round_touched_contexts": round(t_warm * 1e3, 3),
            "gbs": round(moved / t_ours / 1e9, 2),
            "cpu_oracle_ms_1core": round(t_ref * 1e3, 2),
            "speedup_vs_cpu": round(t_ref / t_ours, 1),
            "v_bit_exact": bool(same_v), "k_max_abs_err": err_k}


def selection_bench(tk, spec, pool, maps, dev, args, peak):
    """K4 over the round: every agent's shared rows at the check layer (layer
    1, as PicConfig's default) are compared with probe keys in one pass; the
    cached side is read straight from the pool by slot."""
    import torch
    from paper_2604_03143_b200 import select as sel
    check = 1 if spec.num_layers > 1 else 0
    starts = np.stack([rounds_segment_starts(spec, a) for a in range(len(maps))])
    tok = np.arange(spec.seg_len)
    rows = np.concatenate([m.slots[(st[:, None] + tok).reshape(-1)]
                           for m, st in zip(maps, starts)])
    d_rows = torch.from_numpy(rows).to(dev)
    plane = pool.k[check]
    g = torch.Generator(device=dev).manual_seed(5)
    fresh = plane[d_rows].clone()
    fresh += (0.05 * torch.randn(fresh.shape, generator=g, device=dev)).to(fresh.dtype)
    counts = [spec.num_segments * spec.seg_len] * len(maps)
    for _ in range(2):
        out = sel.batched_selection(fresh, plane, counts, 0.15, cached_rows=d_rows)
    reps = max(1, min(args.steps, 5))
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(reps):
        out = sel.batched_selection(fresh, plane, counts, 0.15, cached_rows=d_rows)
    torch.cuda.synchronize(dev)
    t = (time.perf_counter() - t0) / reps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sel.selection_kernels(fresh, plane, d_rows, counts, 0.15)
    e1.record()
    torch.cuda.synchronize(dev)
    tk_s = e0.elapsed_time(e1) * 1e-3 / reps
    nbytes = 2 * fresh.numel() * fresh.element_size() + 4 * len(rows)
    return {"members": len(maps), "rows": int(len(rows)),
            "important_per_member": int(len(out[0][0])),
            "gbs": round(nbytes / t / 1e9, 1), "frac": round(nbytes / t / 1e9 / peak, 4),
            "ms_per_round": round(t * 1e3, 3),
            "device_gbs": round(nbytes / tk_s / 1e9, 1),
            "device_frac": round(nbytes / tk_s / 1e9 / peak, 4),
            "device_ms": round(tk_s * 1e3, 4),
            "bytes": "fresh + cached check-layer rows read once (+ magnitudes); whole API call "
                     "incl. the host read of important sets and deviations"}


def recompute_bench(dev, args):
    """K5: the tensor-core projection GEMM at a Qwen2.5-7B-shaped selective
    recompute (2048 deviating rows x fused QKV 3584 -> 4608), bf16 and
    3xTF32, against the measured bf16 peak; plus the toy model's refresh of
    a C1 round (8 agents) timed against the oracle on the host."""
    import torch
    from paper_2604_03143_b200 import gemm, recompute, rounds
    from oracle import roundkv_port as ref   # CPU timing leg only
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:   # noqa: BLE001
        pass
    bf16_peak = float(peaks.get("bf16_tflops", 1590.0))
    out = {}
    M, N, K = 2048, 4608, 3584
    g = torch.Generator(device=dev).manual_seed(1)
    for name, dt, rounds_ in (("bf16", torch.bfloat16, 20), ("tf32x3", torch.float32, 5)):
        a = torch.randn(M, K, generator=g, device=dev).to(dt)
        b = torch.randn(N, K, generator=g, device=dev).to(dt)
        c = torch.empty(M, N, device=dev)
        gemm.gemm_tn(a, b, out=c)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(rounds_):
            gemm.gemm_tn(a, b, out=c)
        e1.record()
        torch.cuda.synchronize(dev)
        t = e0.elapsed_time(e1) * 1e-3 / rounds_
        tflops = 2.0 * M * N * K / t / 1e12
        out[f"gemm_{name}"] = {"shape": [M, N, K], "ms": round(t * 1e3, 4),
                               "tflops": round(tflops, 1),
                               "frac_of_bf16_peak": round(tflops / bf16_peak, 4)}
        if dt == torch.float32:
            # 3xTF32 over pre-split operands: the weights (B) split once, the
            # activations (A) split per GEMM -- the split is inside the timing
            bs = gemm.tf32_split(b)
            asp = (torch.empty_like(a), torch.empty_like(a))
            gemm.tf32_split(a, out=asp)
            gemm.gemm_tf32x3(asp, bs, out=c)
            e0.record()
            for _ in range(rounds_):
                gemm.tf32_split(a, out=asp)
                gemm.gemm_tf32x3(asp, bs, out=c)
            e1.record()
            torch.cuda.synchronize(dev)
            t = e0.elapsed_time(e1) * 1e-3 / rounds_
            tflops = 2.0 * M * N * K / t / 1e12
            out["gemm_tf32x3_presplit"] = {
                "shape": [M, N, K], "ms": round(t * 1e3, 4), "tflops": round(tflops, 1),
                "frac_of_bf16_peak": round(tflops / bf16_peak, 4),
                "note": "tdkv_tf32_split of A + tdkv_gemm_tf32x3 (B split once, like weights)"}
    # toy-model refresh of a C1-shaped round (L=2, H=8, D=64), 8 agents;
    # synthetic weights from the product's generator, handed to the oracle
    # only for its CPU timing leg
    _W = rounds.toy_weights(2, 8, 64, 1024, seed=0)
    w = ref.ToyWeights(8, 64, 10000.0, _W.embed, _W.wq, _W.wk, _W.wv, _W.wm)
    rng = np.random.default_rng(3)
    T = 1092
    toks = rng.integers(0, 1023, T)
    ctx_k = rng.standard_normal((2, T, 8, 64)).astype(np.float32) * 0.1
    ctx_v = rng.standard_normal((2, T, 8, 64)).astype(np.float32) * 0.1
    fixes = [np.union1d(np.sort(rng.choice(np.arange(65, T), 154, replace=False)),
                        [64, 321, 578, 835]).astype(np.int64) for _ in range(8)]
    dk, dv = torch.from_numpy(ctx_k).to(dev), torch.from_numpy(ctx_v).to(dev)
    pos = np.arange(T, dtype=np.int64)
    for f in fixes[:2]:
        recompute.selective_forward(_W, toks, pos, f, dk, dv)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for f in fixes:
        recompute.selective_forward(_W, toks, pos, f, dk, dv)
    torch.cuda.synchronize(dev)
    gpu_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    for f in fixes[:2]:
        ref.selective_forward(w, toks, pos, f, ctx_k, ctx_v)
    cpu_s = (time.perf_counter() - t0) * len(fixes) / 2
    out["toy_refresh_c1"] = {"agents": 8, "rows_per_agent": int(fixes[0].size),
                             "gpu_ms": round(gpu_s * 1e3, 3),
                             "cpu_oracle_ms_1core": round(cpu_s * 1e3, 1),
                             "speedup": round(cpu_s / gpu_s, 1)}
    return out


def recovery_bench(dev, args):
    """The Collector's caller, end to end on the GPU: grouped recovery
    (collective_recover: one Collector pass, one selection pass, per-member
    refresh, master election, mirror hints) vs serial recover_prepared of every
    member, on BASELINE configs[0] (8 agents x 4 shared 256-token blocks,
    2-layer toy model, 8 heads, d=64; synthetic weights and tokens) -- the
    paper's collective-vs-serial PIC comparison."""
    import torch
    from paper_2604_03143_b200 import pic, rounds
    from paper_2604_03143_b200.ledger import CostLedger

    class _Pic:
        recompute_fraction = 0.15
        check_layer = 1
    w = rounds.toy_weights(2, 8, 64, 1024, seed=0)
    members = rounds.toy_round(w, seed=1, device=dev)     # segment masters resident in HBM
    group = rounds.ToyGroup(members)

    def grouped():
        led = CostLedger(2)
        pic.collective_recover(w, group, _Pic, led)
        return led

    def serial():
        led = CostLedger(2)
        for m in members:
            pic.recover_prepared(w, m, _Pic, led)
        return led

    out = {"agents": len(members), "tokens_per_agent": int(members[0].num_tokens)}
    torch.cuda.empty_cache()         # the codec sub-benchmarks leave large cached blocks
    for name, fn in (("grouped", grouped), ("serial", serial)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        times = []
        for _ in range(11):
            t0 = time.perf_counter()
            led = fn()
            torch.cuda.synchronize(dev)
            times.append(time.perf_counter() - t0)
        out[f"{name}_ms"] = round(float(np.median(times)) * 1e3, 3)
        out[f"{name}_ms_min"] = round(float(np.min(times)) * 1e3, 3)
        out[f"{name}_rope_calls_per_layer"] = led.rope_calls_per_layer
        out[f"{name}_selection_passes"] = led.selection_passes
    out["speedup"] = round(out["serial_ms"] / out["grouped_ms"], 2)
    out["agents_per_s"] = round(len(members) / (out["grouped_ms"] * 1e-3), 1)
    # group-size sweep, as the paper's Q2 (3 / 5 / 10 / 15 / 20 agents)
    sweep = []
    for n in (3, 5, 10, 15, 20):
        mem = rounds.toy_round(w, num_agents=n, seed=2, device=dev)
        grp = rounds.ToyGroup(mem)
        row = {"agents": n}
        for name, fn in (("grouped", lambda: pic.collective_recover(w, grp, _Pic)),
                         ("serial", lambda: [pic.recover_prepared(w, x, _Pic) for x in mem])):
            fn()
            torch.cuda.synchronize(dev)
            times = []
            for _ in range(5):
                t0 = time.perf_counter()
                fn()
                torch.cuda.synchronize(dev)
                times.append(time.perf_counter() - t0)
            row[f"{name}_ms"] = round(float(np.median(times)) * 1e3, 3)
        row["speedup"] = round(row["serial_ms"] / row["grouped_ms"], 2)
        sweep.append(row)
    out["group_size_sweep"] = sweep
    out["note"] = ("wall clock (median of 11) incl. host control flow and the selection "
                   "read-back; segment masters resident in HBM; the paper reports up to 2.57x "
                   "collective over serial on A100 + vLLM")
    return out


def rounds_segment_starts(spec, a):
    from paper_2604_03143_b200 import rounds
    return rounds.segment_starts(spec, a)


def codec_sweep(tk, spec, pool, maps, dev, args, peak):
    """The diff-aware storage sweep of SURVEY §8d: changed-block fractions
    0 .. 1, the natural AgentSociety fraction (the 8,192 private of 12,320
    rows differ: ~0.66 of the blocks), plus the 'hint everything' variant at 10%."""
    out = []
    for frac, hint_all in ((0.0, False), (0.05, False), (0.1, False), (0.2, False),
                           (0.5, False), (0.66, False), (1.0, False), (0.1, True)):
        r = codec_bench(tk, spec, pool, maps, dev, args, peak, frac=frac, hint_all=hint_all)
        out.append({"changed_fraction": frac, "hint_all": hint_all,
                    "encode_gbs": r["encode_gbs"], "encode_device_gbs": r["encode_device_gbs"],
                    "decode_gbs": r["decode_gbs"], "compression_ratio": r["compression_ratio_mean"]})
        torch_empty_cache()
    return out


def torch_empty_cache():
    import torch
    torch.cuda.empty_cache()


def codec_bench(tk, spec, pool, maps, dev, args, peak, frac=None, hint_all=False):
    """Encode the agents' caches as diffs against agent 0's, then fused-restore
    every mirror into the pool; each mirror is agent 0's cache with a
    fraction of its 32-token blocks (all layers) re-drawn."""
    import torch
    bs = 32
    T = spec.tokens_per_agent
    nb = -(-T // bs)
    frac = args.mirror_frac if frac is None else frac
    # a family is one session (trace.py:365-386: one family per group): at
    # C3 the master and the other 24 agents of its session
    per_family = spec.agents_per_session if spec.sessions > 1 else len(maps)
    n_mirrors = max(1, min(len(maps) - 1, per_family - 1, args.codec_mirrors))
    sl0 = maps[0].device_slots(dev)
    mk = pool.k[:, sl0].contiguous()
    mv = pool.v[:, sl0].contiguous()
    master = tk.LayeredKv(mk, mv, np.arange(T))
    rng = np.random.default_rng(3)
    g = torch.Generator(device=dev).manual_seed(3)
    mirrors, hints = [], []
    n_pick = int(round(frac * nb))
    tok_block = torch.arange(T, device=dev) // bs
    for _ in range(n_mirrors):
        blocks = np.sort(rng.choice(nb, n_pick, replace=False))
        sel = torch.zeros(nb, dtype=torch.bool, device=dev)
        if n_pick:
            sel[torch.from_numpy(blocks).to(dev)] = True
        row = sel[tok_block].view(1, T, 1, 1)
        k = torch.where(row, torch.randn(mk.shape, generator=g, device=dev).to(mk.dtype), mk)
        v = torch.where(row, torch.randn(mv.shape, generator=g, device=dev).to(mv.dtype), mv)
        mirrors.append(tk.LayeredKv(k, v, np.arange(T)))
        if hint_all:
            hints.append(np.arange(T))
        else:
            hints.append(np.concatenate([np.arange(b * bs, min(T, b * bs + bs)) for b in blocks])
                         if n_pick else np.zeros(0, np.int64))
    blocks_cfg = tk.CacheBlockConfig(bs)
    dense = spec.dense_bytes
    # encode (K2 compare + compact + the host read of counts/indices)
    for _ in range(2):
        diffs = tk.encode_batch(master, mirrors, hints, blocks_cfg)
    torch.cuda.synchronize(dev)
    reps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(reps):
        diffs = None
        diffs = tk.encode_batch(master, mirrors, hints, blocks_cfg)
    torch.cuda.synchronize(dev)
    enc_s = (time.perf_counter() - t0) / reps
    # the two K2 launches alone (CUDA events; descriptor upload included)
    from paper_2604_03143_b200 import diffstore as _ds
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = _ds.encode_launch(master, mirrors, hints, blocks_cfg)
    torch.cuda.synchronize(dev)
    # device-timed loops run 20 back-to-back calls: the first call's host
    # submission (GPU idle before its launch) is amortized as in a stream of
    # families; later calls' submissions overlap the previous launch
    dreps = max(reps, 20)
    e0.record()
    for _ in range(dreps):
        st = None    # release the previous outputs so the caching allocator reuses them
        st = _ds.encode_launch(master, mirrors, hints, blocks_cfg)
    e1.record()
    torch.cuda.synchronize(dev)
    enc_dev_s = e0.elapsed_time(e1) * 1e-3 / dreps
    del st
    payload = sum(d.payload_nbytes for d in diffs)
    changed = sum(sum(d.changed_blocks_per_layer) for d in diffs)
    enc_bytes = n_mirrors * 2 * dense + payload + 4 * changed
    # the family byte model: the master is read once for the whole family
    # (K2/K3 order their work so the P mirrors of a master tile run back to
    # back and share it through L2)
    enc_family_bytes = dense + n_mirrors * dense + payload + 4 * changed
    # fused restore of every mirror into its agent's slots
    fam = tk.MasterEntry(0, master, pin_count=n_mirrors)
    handles = [tk.MirrorHandle(0, i + 1, fam, d) for i, d in enumerate(diffs)]
    spans = [tk.PositionSpan.shifted(np.arange(T), 16) for _ in handles]
    tmaps = maps[1:1 + n_mirrors]
    for _ in range(2):
        tk.fused_restore_many(handles, spans, pool, tmaps, 10000.0)
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(dreps):
        tk.fused_restore_many(handles, spans, pool, tmaps, 10000.0)
    ev1.record()
    torch.cuda.synchronize(dev)
    dec_s = ev0.elapsed_time(ev1) * 1e-3 / dreps
    dec_bytes = n_mirrors * 2 * dense
    dec_family_bytes = dense + payload + n_mirrors * dense
    # the paper's fused-vs-dense comparison, one mirror per
    # API call as the reference restores them (trace.py:314-318): fused_restore
    # vs dense_restore (materialize the mirror, then rotate + write it)
    per = {}
    for name, fn in (("fused", tk.fused_restore), ("dense", tk.dense_restore)):
        for h, sp, m in zip(handles[:2], spans, tmaps):
            fn(h, sp, pool, m, 10000.0)
        torch.cuda.synchronize(dev)
        ev0.record()
        for h, sp, m in zip(handles, spans, tmaps):
            fn(h, sp, pool, m, 10000.0)
        ev1.record()
        torch.cuda.synchronize(dev)
        per[name] = ev0.elapsed_time(ev1) / n_mirrors
    wire = [tk.wire_nbytes(d) for d in diffs]       # == len(serialize_diff(d))
    dense_f32 = tk.kv_dense_nbytes(T, spec.num_layers, spec.num_heads, spec.head_dim)
    pay_bytes = [d.payload_nbytes for d in diffs]
    # TDDF wire images (float32 payload, the reference format): GPU pack of
    # the whole family + one D2H, and GPU unpack of one image into device
    # slabs (H2D included); bytes = wire image bytes
    # one untimed call of each first: it pins the host staging buffers,
    # which torch's caching host allocator then reuses
    images = tk.serialize_many(diffs, copy=False)
    for w in images[:8]:
        tk.deserialize_to_device(w, dev, pool.k.dtype)
    torch.cuda.synchronize(dev)
    del images, w        # the views pin the staging buffer: release it for reuse
    t0 = time.perf_counter()
    images = tk.serialize_many(diffs, copy=False)
    pack_s = time.perf_counter() - t0
    wire_total = sum(len(w) for w in images)
    t0 = time.perf_counter()
    for w in images[:8]:
        tk.deserialize_to_device(w, dev, pool.k.dtype)
    torch.cuda.synchronize(dev)
    unpack_s = time.perf_counter() - t0
    unpack_bytes = sum(len(w) for w in images[:8])
    # the same images as Python bytes objects (pageable: what a reader of
    # files / sockets holds) -- staged through the pinned ring
    owned = [bytes(w) for w in images[:8]]
    del images
    for w in owned[:2]:               # both pinned ring buffers allocated
        tk.deserialize_to_device(w, dev, pool.k.dtype)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for w in owned:
        tk.deserialize_to_device(w, dev, pool.k.dtype)
    torch.cuda.synchronize(dev)
    unpack_bytes_s = time.perf_counter() - t0
    del owned
    return {
        "mirrors": n_mirrors, "changed_block_fraction": round(changed / (n_mirrors * spec.num_layers * nb), 4),
        "encode_gbs": round(enc_bytes / enc_s / 1e9, 1),
        "encode_frac": round(enc_bytes / enc_s / 1e9 / peak, 4),
        "encode_ms_per_family": round(enc_s * 1e3, 3),
        "encode_device_gbs": round(enc_bytes / enc_dev_s / 1e9, 1),
        "encode_device_frac": round(enc_bytes / enc_dev_s / 1e9 / peak, 4),
        "decode_gbs": round(dec_bytes / dec_s / 1e9, 1),
        "decode_frac": round(dec_bytes / dec_s / 1e9 / peak, 4),
        "decode_ms_per_family": round(dec_s * 1e3, 3),
        "family_model": {
            "encode_bytes": int(enc_family_bytes), "decode_bytes": int(dec_family_bytes),
            "encode_device_gbs": round(enc_family_bytes / enc_dev_s / 1e9, 1),
            "encode_device_frac": round(enc_family_bytes / enc_dev_s / 1e9 / peak, 4),
            "decode_gbs": round(dec_family_bytes / dec_s / 1e9, 1),
            "decode_frac": round(dec_family_bytes / dec_s / 1e9 / peak, 4),
            "bytes": "encode: dense (master once) + P*dense (mirrors) + payload + 4*changed; "
                     "decode: dense (master once) + payload + P*dense (pool writes)"},
        "restore_ms_per_mirror": {"fused": round(per["fused"], 4), "dense": round(per["dense"], 4),
                                  "dense_over_fused": round(per["dense"] / per["fused"], 2),
                                  "note": "one mirror per API call (host planning included), "
                                          f"CUDA events around the {n_mirrors} calls"},
        # CompressionStats.ratios as the reference computes them: float32 dense
        # bytes / bytes of the float32 TDDF image serialize_diff emits
        "compression_ratio_mean": round(float(np.mean([dense_f32 / w for w in wire])), 3),
        # the in-HBM form: bf16 dense cache / bf16 payload slab bytes
        "payload_ratio_mean": round(float(np.mean([dense / max(1, b) for b in pay_bytes])), 3),
        "wire_pack_gbs": round(wire_total / pack_s / 1e9, 2),
        "wire_unpack_gbs": round(unpack_bytes / unpack_s / 1e9, 2),
        "wire_unpack_pageable_gbs": round(unpack_bytes / unpack_bytes_s / 1e9, 2),
        "wire_note": "serialize_many of the family (GPU pack, one D2H into pinned memory, "
                     "images as memoryviews) and "
                     "deserialize_to_device of 8 images (host parse, one H2D each, GPU "
                     "unpack): wire_unpack_gbs from those pinned views (H2D straight from "
                     "them), wire_unpack_pageable_gbs from bytes copies of them (host threads "
                     "stage each into a pinned ring buffer); wall clock after one untimed "
                     "call, float32 wire bytes",
        "bytes": "encode: 2*dense + payload + 4*changed per mirror (host read included); "
                 "fused decode: 2*dense per mirror (K0+K3 device time)",
        "timing": f"encode_gbs: {reps} encode_batch calls, wall clock incl. the host read of "
                  f"counts/indices; encode_device / decode: CUDA events around {dreps} "
                  "back-to-back API calls (submission of the first one included)",
    }


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_tdkv(args)


if __name__ == "__main__":
    main()
