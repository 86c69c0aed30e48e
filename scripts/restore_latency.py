"""Per-call latency of fused_restore / dense_restore at the C2 mirror shape
(one mirror per API call, as the reference restores them) with a host-side
profile of the fused call (diagnostic)."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_03143_b200 as tk  # noqa: E402

L, T, H, D, bs, P = 28, 4624, 4, 128, 32, 16
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
mk = torch.randn(L, T, H, D, generator=g, device=dev).bfloat16()
mv = torch.randn(L, T, H, D, generator=g, device=dev).bfloat16()
master = tk.LayeredKv(mk, mv, np.arange(T))
nb = -(-T // bs)
rng = np.random.default_rng(1)
mirrors, hints = [], []
for _ in range(P):
    blocks = np.sort(rng.choice(nb, nb // 10, replace=False))
    k = mk.clone()
    for b in blocks:
        k[:, b * bs:(b + 1) * bs] += 1
    mirrors.append(tk.LayeredKv(k, mv, np.arange(T)))
    hints.append(np.concatenate([np.arange(b * bs, min(T, b * bs + bs)) for b in blocks]))
diffs = tk.encode_batch(master, mirrors, hints, tk.CacheBlockConfig(bs))
del mirrors
pool = tk.PagedPool(P * T, L, H, D, dtype=torch.bfloat16, device=dev, debug=False)
maps = [pool.allocate(T, i) for i in range(P)]
fam = tk.MasterEntry(0, master, pin_count=P)
handles = [tk.MirrorHandle(0, i + 1, fam, d) for i, d in enumerate(diffs)]
spans = [tk.PositionSpan.shifted(np.arange(T), 16) for _ in handles]
for name, fn in (("fused", tk.fused_restore), ("dense", tk.dense_restore)):
    for h, sp, m in zip(handles, spans, maps):
        fn(h, sp, pool, m, 10000.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for h, sp, m in zip(handles, spans, maps):
        fn(h, sp, pool, m, 10000.0)
    t_host = (time.perf_counter() - t0) / P
    torch.cuda.synchronize()
    t_all = (time.perf_counter() - t0) / P
    print(f"{name}: host {t_host * 1e3:.3f} ms/call, with device {t_all * 1e3:.3f} ms/mirror")
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    for h, sp, m in zip(handles, spans, maps):
        tk.fused_restore(h, sp, pool, m, 10000.0)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
