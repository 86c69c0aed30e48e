"""A/B timing of the fused family restore at the C2 codec-bench shape
(TDKV_RESTORE_FAMILY=1: K0 + K1 with the diff overlay; 0: K0 + K3):
run once per library build (TDKV_LIBRARY=...), prints median GB/s of 15
samples of 6 back-to-back 49-mirror family restores (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_03143_b200 as tk  # noqa: E402

# RESTORE_SHAPE=c3: the C3 codec family (one session: 24 mirrors of 717 tokens, L=48, H=8)
L, T, H, D, bs, P = ((48, 717, 8, 128, 32, 24) if os.environ.get("RESTORE_SHAPE") == "c3"
                     else (28, 4624, 4, 128, 32, 49))
P = int(os.environ.get("RESTORE_MIRRORS", P))      # family size override (threshold sweeps)
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
    k, v = mk.clone(), mv.clone()
    for b in blocks:
        k[:, b * bs:(b + 1) * bs] += 1
    mirrors.append(tk.LayeredKv(k, v, np.arange(T)))
    hints.append(np.concatenate([np.arange(b * bs, min(T, b * bs + bs)) for b in blocks]))
del k, v
diffs = tk.encode_batch(master, mirrors, hints, tk.CacheBlockConfig(bs))
del mirrors
pool = tk.PagedPool(P * T + 64, L, H, D, dtype=torch.bfloat16, device=dev, debug=False)
maps = [pool.allocate(T, i) for i in range(P)]
fam = tk.MasterEntry(0, master, pin_count=P)
handles = [tk.MirrorHandle(0, i + 1, fam, d) for i, d in enumerate(diffs)]
spans = [tk.PositionSpan.shifted(np.arange(T), 16) for _ in handles]
for _ in range(3):
    tk.fused_restore_many(handles, spans, pool, maps, 10000.0)
torch.cuda.synchronize()
res = []
for _ in range(5):       # 6 back-to-back restores per sample: host prep overlaps the GPU
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(6):
        tk.fused_restore_many(handles, spans, pool, maps, 10000.0)
    b.record()
    torch.cuda.synchronize()
    res.append(a.elapsed_time(b) * 1e-3 / 6)
import time  # noqa: E402
host = []
for _ in range(7):       # host-side cost of one call (the GPU idle before it)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tk.fused_restore_many(handles, spans, pool, maps, 10000.0)
    host.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print("host ms per call (submission, median of 7)", round(np.median(host) * 1e3, 4))
dense = 2 * L * T * H * D * 2
payload = sum(2 * sum(ld.indices.size for ld in d.layers) * bs * H * D * 2 for d in diffs)
fam_bytes = dense + payload + P * dense
print("family model GB/s median", round(fam_bytes / np.median(res) / 1e9, 1),
      "ms", round(np.median(res) * 1e3, 4))
print(os.environ.get("TDKV_LIBRARY", "in-tree"), "fused restore GB/s median",
      round(P * 2 * dense / np.median(res) / 1e9, 1), "best", round(P * 2 * dense / min(res) / 1e9, 1))
