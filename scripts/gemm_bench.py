"""tdkv_gemm variants vs cuBLAS (torch.matmul) on a few shapes (diagnostic).

Prints TFLOP/s for: the CTA-pair kernel (default for large shapes), the
single-CTA persistent kernel (TDKV_GEMM_NO_PAIR=1), the non-persistent TMA
kernel (+ TDKV_GEMM_NO_PERSISTENT=1), and cuBLAS via torch.matmul (bf16 out)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_03143_b200 import gemm  # noqa: E402


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e-3 / reps


for M, N, K in [(2048, 4608, 3584), (2048, 3584, 3584), (4096, 4096, 4096), (8192, 8192, 8192)]:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda")
    fl = 2.0 * M * N * K
    row = [f"{M}x{N}x{K}"]
    for mode, env in (("pair", {}), ("persistent", {"TDKV_GEMM_NO_PAIR": "1"}),
                      ("tma", {"TDKV_GEMM_NO_PAIR": "1", "TDKV_GEMM_NO_PERSISTENT": "1"})):
        for key in ("TDKV_GEMM_NO_PAIR", "TDKV_GEMM_NO_PERSISTENT"):
            os.environ.pop(key, None)
        os.environ.update(env)
        t = timeit(lambda: gemm.gemm_tn(a, b, out=c))
        row.append(f"{mode} {fl / t / 1e12:.0f}")
    for key in ("TDKV_GEMM_NO_PAIR", "TDKV_GEMM_NO_PERSISTENT"):
        os.environ.pop(key, None)
    t = timeit(lambda: torch.matmul(a, b.T))
    row.append(f"cublas(bf16 out) {fl / t / 1e12:.0f}")
    print("  ".join(row), flush=True)
