#!/usr/bin/env python
"""Direction-resolved HBM ceilings on this B200 (context for the rooflines;
the reported denominator stays MEASURED_PEAKS.json's copy figure).

Read-only: torch.sum over 8 GiB; write-only: fill_; copy: copy_ (read+write).
CUDA events, best of 10.
"""
import json

import torch


def best(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e-3)
    return min(out)


def main():
    n = 4 << 30            # 4 Gi bf16 elements = 8 GiB
    x = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
    y = torch.empty_like(x)
    nbytes = x.numel() * 2
    r = best(lambda: x.sum(dtype=torch.float32))
    w = best(lambda: y.fill_(1.0))
    c = best(lambda: y.copy_(x))
    print(json.dumps({"read_gbs": round(nbytes / r / 1e9, 1), "write_gbs": round(nbytes / w / 1e9, 1),
                      "copy_gbs": round(2 * nbytes / c / 1e9, 1), "bytes": nbytes}))


if __name__ == "__main__":
    main()
