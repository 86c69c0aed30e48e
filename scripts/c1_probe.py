"""C1 collector timing probe (A/B helper, run under gpurun): one C1 round
(configs[0] shape: 8 agents x 4 shared 256-token blocks, L=2, H=8, D=64, f32)
timed per round with CUDA events under several L2 states:

  write   -- a 2 x L2 buffer written before each round (bench.py's flush)
  wread   -- the same, then a 2 x L2 buffer read (the flush's dirty lines
             written back before the round starts)
  warm    -- rounds back to back, no flush (output and masters L2-resident)

Env knobs of the plan (TDKV_PLAN_ITEMS, TDKV_TILE_SMEM, TDKV_FUSE_TABLE) are
read at import, so A/B runs use separate processes.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_03143_b200 as tk  # noqa: E402
from paper_2604_03143_b200 import rounds  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    spec = rounds.CONFIGS[cfg]
    dt = spec.torch_dtype
    mk, mv = rounds.master_planes_host(spec)
    arena = rounds.make_arena(spec, torch.from_numpy(mk).to(dt).to(dev),
                              torch.from_numpy(mv).to(dt).to(dev))
    T = spec.tokens_per_agent
    pool = tk.PagedPool(spec.num_agents * T, spec.num_layers, spec.num_heads, spec.head_dim,
                        dtype=dt, device=dev, debug=False)
    maps = [pool.allocate(T, a) for a in range(spec.num_agents)]
    col = tk.KVCollector(arena, pool)
    plan = col.plan([j for a in range(spec.num_agents)
                     for j in rounds.agent_jobs(spec, a, maps[a].slots)])
    nbytes = plan.algorithmic_bytes()
    l2 = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 0) or 126 * 2**20)
    wbuf = torch.empty(2 * l2, dtype=torch.uint8, device=dev)
    rbuf = torch.ones(2 * l2 // 4, dtype=torch.float32, device=dev)
    sink = torch.empty(1, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    out = {"config": cfg, "bytes": nbytes, "units": int(plan.units_host.size),
           "tile_rows": int(plan.tile_rows), "fuse_table": bool(plan.fuse_table)}
    for mode in ("write", "wread", "warm"):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(reps)]
        for i in range(reps + 5):
            if mode != "warm":
                wbuf.fill_(1)
            if mode == "wread":
                sink.copy_(rbuf.sum())
            if i >= 5:
                ev[i - 5][0].record(stream)
            col.collect(plan)
            if i >= 5:
                ev[i - 5][1].record(stream)
        torch.cuda.synchronize(dev)
        us = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
        out[mode] = {"us_median": round(float(np.median(us)), 2),
                     "us_min": round(float(us.min()), 2),
                     "us_mean": round(float(us.mean()), 2),
                     "gbs_mean": round(nbytes / (us.mean() * 1e-6) / 1e9, 1)}
    # back to back, one event pair around all rounds
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        col.collect(plan)
    b.record(stream)
    torch.cuda.synchronize(dev)
    us = a.elapsed_time(b) * 1e3 / reps
    out["b2b"] = {"us": round(us, 2), "gbs": round(nbytes / (us * 1e-6) / 1e9, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
