"""Split deserialize_to_device's wall time at C2 image sizes: structural
parse, staging (host threads fill pinned chunks + chunked H2D), the unpack
launch, and the whole call (python scripts/wire_host_profile.py)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_03143_b200 as tk  # noqa: E402
from paper_2604_03143_b200 import _device, diffstore  # noqa: E402

DEV = torch.device("cuda", 0)
rng = np.random.default_rng(0)
t, L, H, D, bs = 4624, 28, 4, 128, 32          # a C2 mirror: 10% of blocks changed
k = rng.standard_normal((L, t, H, D)).astype(np.float32)
master = tk.LayeredKv(torch.from_numpy(k).to(DEV).bfloat16(), torch.from_numpy(k).to(DEV).bfloat16(),
                      np.arange(t))
nb = -(-t // bs)
mirrors, hints = [], []
for _ in range(8):
    ids = np.sort(rng.choice(nb, nb // 10, replace=False))
    mk = master.k.clone()
    for b in ids:
        mk[:, b * bs:(b + 1) * bs] += 1
    mirrors.append(tk.LayeredKv(mk, master.v.clone(), master.positions))
    hints.append((ids[:, None] * bs + np.arange(bs)).reshape(-1))
diffs = tk.encode_batch(master, mirrors, hints, tk.CacheBlockConfig(bs))
views = tk.serialize_many(diffs, copy=False)
owned = [bytes(v) for v in views]
print("image MB", len(owned[0]) / 1e6)


def timed(fn, reps=8):
    ts = []
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(r)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3


for name, imgs in (("pinned views", views), ("bytes", owned)):
    n = len(imgs[0])
    print(name)
    print("  parse ms", timed(lambda r: diffstore._parse_wire(imgs[r % 8])))
    print("  stage ms", timed(lambda r: _device.bytes_to_device(imgs[r % 8], DEV, 8)),
          "(PCIe alone %.2f ms at 55 GB/s)" % (n / 55e6))
    print("  whole ms", timed(lambda r: tk.deserialize_to_device(imgs[r % 8], DEV, torch.bfloat16)))
    src = np.frombuffer(imgs[0], np.uint8)
    dst = np.empty(n, np.uint8)
    print("  one-thread memcpy ms", timed(lambda r: dst.__setitem__(slice(None), src)))
