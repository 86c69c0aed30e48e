"""Where the K4 API time goes at the C3 round shape (diagnostic, under gpurun):
host submission, device time, read-back + sync, host unpacking."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_03143_b200 import select as sel  # noqa: E402

dev = torch.device("cuda", 0)
M, N, H, D = 250, 500, 8, 128
g = torch.Generator(device=dev).manual_seed(0)
plane = torch.randn(M * N * 2, H, D, generator=g, device=dev).bfloat16()
rows = torch.arange(M * N, device=dev) * 2
fresh = (plane[rows].float() + 0.05 * torch.randn(M * N, H, D, generator=g, device=dev)).bfloat16()
counts = [N] * M
for _ in range(3):
    sel.batched_selection(fresh, plane, counts, 0.15, cached_rows=rows)
torch.cuda.synchronize()
T = {"api": [], "submit": [], "device+readback": [], "unpack": []}
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sel.batched_selection(fresh, plane, counts, 0.15, cached_rows=rows)
    T["api"].append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    off, buf = sel.selection_kernels(fresh, plane, rows, counts, 0.15)
    t1 = time.perf_counter()
    staged = torch.empty(buf.shape, dtype=buf.dtype, pin_memory=True)
    staged.copy_(buf, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    t2 = time.perf_counter()
    host = staged.numpy()
    cnt_h = host[:M].tolist()
    sums = host[M:2 * M].view(np.float32).tolist()
    idx_h = host[2 * M:].astype(np.int64)
    starts = off.tolist()
    out = [(idx_h[starts[i]:starts[i] + cnt_h[i]], sums[i]) for i in range(M)]
    t3 = time.perf_counter()
    T["submit"].append(t1 - t0)
    T["device+readback"].append(t2 - t1)
    T["unpack"].append(t3 - t2)
print({k: round(float(np.median(v)) * 1e6, 1) for k, v in T.items()}, "us (median of 50)")
