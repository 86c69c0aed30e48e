import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2604_03143_b200 import _device, _lib
DEV = torch.device("cuda", 0)
n = 51_381_960
srcs = [bytes(np.random.bytes(n)) for _ in range(8)]
_device.bytes_to_device(srcs[0], DEV, 8); _device.bytes_to_device(srcs[1], DEV, 8)
torch.cuda.synchronize()
lib = _lib.load()
for it in range(6):
    buf = srcs[it % 8]
    T = [time.perf_counter()]
    src = np.frombuffer(buf, np.uint8); T.append(time.perf_counter())
    out = torch.empty(n + 8, dtype=torch.uint8, device=DEV); T.append(time.perf_counter())
    p = lib.tdkv_host_is_pinned(src.ctypes.data); T.append(time.perf_counter())
    st = _device._stage_rings[DEV][0][0]
    sv = st.buf.numpy(); T.append(time.perf_counter())
    bounds = list(range(0, n, 2 << 20)) + [n]
    def fill(c):
        sv[bounds[c]:bounds[c + 1]] = src[bounds[c]:bounds[c + 1]]
    list(_device.host_executor().map(fill, range(len(bounds) - 1))); T.append(time.perf_counter())
    out.copy_(st.buf[:n + 8], non_blocking=True); T.append(time.perf_counter())
    torch.cuda.synchronize(); T.append(time.perf_counter())
    print("pinned?", p, " ".join("%.3f" % ((b - a) * 1e3) for a, b in zip(T, T[1:])))
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _device.bytes_to_device(srcs[it % 8], DEV, 8); t1 = time.perf_counter(); torch.cuda.synchronize()
    print("b2d call %.3f total %.3f" % ((t1 - t0) * 1e3, (time.perf_counter() - t0) * 1e3))
