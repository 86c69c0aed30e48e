"""Split one encode_batch call into host prep / device / readback phases
(diagnostic for the API-vs-device gap of the encoder)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2604_03143_b200 as tk
from paper_2604_03143_b200 import diffstore as ds

L, T, H, D, bs, P = 28, 8192 + 4096 + 512, 4, 128, 32, 32
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
mk = torch.randn(L, T, H, D, generator=g, device=dev).bfloat16()
mv = torch.randn(L, T, H, D, generator=g, device=dev).bfloat16()
master = tk.LayeredKv(mk, mv, np.arange(T))
nb = -(-T // bs)
for frac in (0.1, 1.0):
    rng = np.random.default_rng(1)
    mirrors, hints = [], []
    for _ in range(P):
        blocks = np.sort(rng.choice(nb, int(frac * nb), replace=False))
        k, v = mk.clone(), mv.clone()
        for b in blocks[:64]:
            k[:, b * bs] += 1
        mirrors.append(tk.LayeredKv(k, v, np.arange(T)))
        hints.append(np.concatenate([np.arange(b * bs, min(T, b * bs + bs)) for b in blocks]))
    cfg = tk.CacheBlockConfig(bs)
    for _ in range(3):
        d = None
        d = ds.encode_batch(master, mirrors, hints, cfg)
    torch.cuda.synchronize()
    t = np.zeros(4)
    for _ in range(5):
        d = None
        t0 = time.perf_counter()
        st = ds.encode_launch(master, mirrors, hints, cfg)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        d = ds.encode_finish(st)
        t3 = time.perf_counter()
        st = None
        t += [t1 - t0, t2 - t1, t3 - t2, t3 - t0]
    t = t / 5 * 1e3
    print(f"frac {frac}: launch(host) {t[0]:.3f} ms  device-wait {t[1]:.3f} ms  finish {t[2]:.3f} ms  total {t[3]:.3f} ms")
