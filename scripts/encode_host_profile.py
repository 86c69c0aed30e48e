"""cProfile of the encoder's host side (encode_launch + encode_finish) at the
C2 codec-bench shape: 49 mirrors, 10% changed blocks (diagnostic)."""
import cProfile
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_03143_b200 as tk  # noqa: E402
from paper_2604_03143_b200 import diffstore as ds  # noqa: E402

import os
# ENCODE_SHAPE=c3: the C3 codec family (24 mirrors of 717 tokens, L=48, H=8)
L, T, H, D, bs, P = ((48, 717, 8, 128, 32, 24) if os.environ.get("ENCODE_SHAPE") == "c3"
                     else (28, 4624, 4, 128, 32, 49))
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
    mirrors.append(tk.LayeredKv(mk.clone(), mv.clone(), np.arange(T)))  # own positions
    hints.append(np.concatenate([np.arange(b * bs, min(T, b * bs + bs)) for b in blocks]))
cfg = tk.CacheBlockConfig(bs)
for _ in range(3):
    ds.encode_batch(master, mirrors, hints, cfg)
torch.cuda.synchronize()
import time  # noqa: E402
host = []
for _ in range(7):      # submission alone (GPU idle before it)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = ds.encode_launch(master, mirrors, hints, cfg)
    host.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = ds.encode_finish(st)
    host.append(-(time.perf_counter() - t0))
print("encode_launch host ms", round(np.median([h for h in host if h > 0]) * 1e3, 4),
      "encode_finish host ms", round(-np.median([h for h in host if h < 0]) * 1e3, 4))
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    st = ds.encode_launch(master, mirrors, hints, cfg)
    torch.cuda.synchronize()
    d = ds.encode_finish(st)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
