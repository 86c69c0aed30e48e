"""Pinned host -> HBM copy bandwidth on this box (the e2e path's ceiling):
one 1 GiB copy, 7 chunks on one stream, and 2 copy streams (diagnostic)."""
import json
import torch

dev = torch.device("cuda", 0)
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device=dev)
out = {}
for name, parts, streams in (("one_copy", 1, 1), ("chunks7", 7, 1), ("chunks8_2streams", 8, 2)):
    ss = [torch.cuda.Stream(dev) for _ in range(streams)]
    for rep in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step = n // parts
        for i in range(parts):
            s = ss[i % streams]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        for s in ss:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else None
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        out[name] = round(n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
print(json.dumps({"h2d_gbs": out}))
