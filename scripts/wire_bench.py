"""Wire path timing at the C2 codec shape (49 mirrors, ~10% changed blocks):
GPU pack vs the host serializer, GPU unpack vs the host parser (diagnostic)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_03143_b200 as tk  # noqa: E402
from paper_2604_03143_b200 import diffstore  # noqa: E402

L, T, H, D, bs, P = 28, 4624, 4, 128, 32, 49
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
images = tk.serialize_many(diffs, copy=False)     # warm the pinned host cache
del images
t0 = time.perf_counter()
images = tk.serialize_many(diffs, copy=False)
t_pack = time.perf_counter() - t0
t0 = time.perf_counter()
tk.serialize_many(diffs)
t_bytes = time.perf_counter() - t0
nbytes = sum(len(w) for w in images)
t0 = time.perf_counter()
host = [diffstore._serialize_host(d) for d in diffs[:4]]
t_host = (time.perf_counter() - t0) * P / 4
assert host == [bytes(w) for w in images[:4]]
tk.deserialize_to_device(images[0], dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
for w in images[:16]:
    tk.deserialize_to_device(w, dev)
torch.cuda.synchronize()
t_unpack = (time.perf_counter() - t0) * P / 16
t0 = time.perf_counter()
for w in images[:4]:
    tk.deserialize_diff(w)
t_parse = (time.perf_counter() - t0) * P / 4
print(f"family wire {nbytes / 1e9:.2f} GB: GPU pack {nbytes / t_pack / 1e9:.2f} GB/s "
      f"(as Python bytes {nbytes / t_bytes / 1e9:.2f} GB/s) "
      f"(host serializer {nbytes / t_host / 1e9:.2f} GB/s); unpack to device "
      f"{nbytes / t_unpack / 1e9:.2f} GB/s (host parse to numpy {nbytes / t_parse / 1e9:.2f} GB/s)")
