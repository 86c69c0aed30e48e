"""Host -> device staging variants for one 51 MB wire image (a C2 mirror):
fill of pinned chunks by host threads, H2D issued by the caller in chunk
order vs by each worker after its fill (python scripts/stage_probe.py)."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_03143_b200 import _device  # noqa: E402

DEV = torch.device("cuda", 0)
n = 51_381_960
src = bytes(np.random.bytes(n))
s = np.frombuffer(src, np.uint8)
keep = torch.empty(n + 8, dtype=torch.uint8, pin_memory=True)
kv = keep.numpy()
dev = torch.empty(n + 8, dtype=torch.uint8, device=DEV)


def t(f, reps=15):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return "%.3f ms" % (np.median(ts) * 1e3)


print("h2d one", t(lambda: dev.copy_(keep, non_blocking=True)))
for nt in (8, 16):
    pool = ThreadPoolExecutor(nt)
    for C in (1 << 20, 2 << 20, 4 << 20):
        b = list(range(0, n, C)) + [n]
        stream = torch.cuda.current_stream(DEV)

        def f(c):
            kv[b[c]:b[c + 1]] = s[b[c]:b[c + 1]]

        def fill():
            list(pool.map(f, range(len(b) - 1)))

        def ordered():
            futs = [pool.submit(f, c) for c in range(len(b) - 1)]
            for c, fu in enumerate(futs):
                fu.result()
                dev[b[c]:b[c + 1]].copy_(keep[b[c]:b[c + 1]], non_blocking=True)

        def g(c):
            kv[b[c]:b[c + 1]] = s[b[c]:b[c + 1]]
            with torch.cuda.stream(stream):
                dev[b[c]:b[c + 1]].copy_(keep[b[c]:b[c + 1]], non_blocking=True)

        def worker_issued():
            list(pool.map(g, range(len(b) - 1)))

        print(nt, "threads", C >> 20, "MB: fill", t(fill), "ordered", t(ordered),
              "worker-issued", t(worker_issued))
print("bytes_to_device", t(lambda: _device.bytes_to_device(src, DEV, 8)))

# cold sources: eight different images cycled (none cache-resident)
srcs = [np.frombuffer(bytes(np.random.bytes(n)), np.uint8) for _ in range(8)]
k = [0]
for nt in (1, 4, 8, 16):
    pool = ThreadPoolExecutor(nt)
    b = list(range(0, n, 2 << 20)) + [n]

    def fc(c):
        sv = srcs[k[0] % 8]
        kv[b[c]:b[c + 1]] = sv[b[c]:b[c + 1]]

    def fill_cold():
        k[0] += 1
        list(pool.map(fc, range(len(b) - 1)))

    print(nt, "threads cold-source fill", t(fill_cold, 16))
print("bytes_to_device cold", t(lambda: _device.bytes_to_device(srcs[k.__setitem__(0, k[0] + 1) or k[0] % 8], DEV, 8), 16))
