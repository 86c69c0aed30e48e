"""K4 diagnostic at the C2 round shape (50 members x 4096 check-layer rows,
bf16 H=4 D=128, cached rows gathered from a pool plane by slot): the
selection_kernels API (tdkv_keydiff + tdkv_select_important, descriptors
uploaded per call) vs the two launches on pre-uploaded descriptors; device
time with CUDA events around back-to-back passes."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_03143_b200 import select as sel  # noqa: E402

dev = torch.device("cuda:0")
M, N, H, D = 50, 4096, 4, 128
if len(sys.argv) > 2:
    M, N = int(sys.argv[1]), int(sys.argv[2])
FRAC = float(sys.argv[3]) if len(sys.argv) > 3 else 0.15
g = torch.Generator(device=dev).manual_seed(0)
plane = torch.randn(M * N + 1000, H, D, generator=g, device=dev).bfloat16()
rows = torch.randperm(M * N + 1000, generator=g, device=dev)[:M * N]
fresh = (plane[rows].float() + 0.05 * torch.randn(M * N, H, D, generator=g, device=dev)).bfloat16()
counts = [N] * M
budgets = [sel.recompute_budget(FRAC, n) for n in counts]
nbytes = 2 * fresh.numel() * 2 + 8 * M * N


def api():
    sel.selection_kernels(fresh, plane, rows, counts, FRAC)


off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
d_off = torch.from_numpy(off).to(dev)
d_bud = torch.from_numpy(np.asarray(budgets, np.int32)).to(dev)
buf = torch.empty(2 * M + M * N, dtype=torch.int32, device=dev)


def two():
    mags = sel._mags_device(fresh, plane, rows)
    sel._lib.call("tdkv_select_important", sel.ptr(mags), sel.ptr(d_off), sel.ptr(d_bud), 0, M, N,
                  sel.ptr(buf) + 8 * M, sel.ptr(buf), sel.ptr(buf) + 4 * M,
                  sel.stream_handle(dev))


for name, fn in (("selection_kernels", api), ("direct", two)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"M={M} N={N} frac={FRAC} {name}: {ms * 1e3:.1f} us, {nbytes / ms / 1e6:.0f} GB/s")

# keydiff alone (the gather-read half of K4)
for _ in range(3):
    sel._mags_device(fresh, plane, rows)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    sel._mags_device(fresh, plane, rows)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"M={M} N={N} keydiff: {ms * 1e3:.1f} us, {nbytes / ms / 1e6:.0f} GB/s")
