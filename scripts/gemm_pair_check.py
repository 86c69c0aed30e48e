"""Correctness + speed of the CTA-pair GEMM (TDKV_GEMM_PAIR=1) on a few shapes."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_03143_b200 import gemm  # noqa: E402

os.environ["TDKV_GEMM_PAIR"] = "1"
for M, N, K in [(256, 256, 64), (300, 512, 512), (2048, 4608, 256), (129, 257, 1000),
                (1000, 1000, 192), (2048, 4608, 3584), (8192, 8192, 8192)]:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    out = gemm.gemm_tn(a, b)
    torch.cuda.synchronize()
    want = a.double() @ b.double().T
    err = (out.double() - want).abs().max().item() / max(1.0, want.abs().max().item())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        gemm.gemm_tn(a, b, out=out)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3 / 10
    print(f"{M}x{N}x{K} relerr {err:.2e} tflops {2.0 * M * N * K / t / 1e12:.0f}", flush=True)
