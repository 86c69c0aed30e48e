"""tdkv_gemm variants vs cuBLAS (torch.matmul) on a few shapes (diagnostic).

Prints TFLOP/s for: persistent TMEM-double-buffered kernel (default), the
non-persistent TMA kernel (TDKV_GEMM_NO_PERSISTENT=1), and torch bf16 matmul
with float32 output semantics (bf16 in, fp32 out via out_dtype)."""
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
    for mode in ("persistent", "tma"):
        if mode == "tma":
            os.environ["TDKV_GEMM_NO_PERSISTENT"] = "1"
        else:
            os.environ.pop("TDKV_GEMM_NO_PERSISTENT", None)
        t = timeit(lambda: gemm.gemm_tn(a, b, out=c))
        row.append(f"{mode} {fl / t / 1e12:.0f}")
    os.environ.pop("TDKV_GEMM_NO_PERSISTENT", None)
    t = timeit(lambda: torch.matmul(a, b.T))
    row.append(f"cublas(bf16 out) {fl / t / 1e12:.0f}")
    print("  ".join(row), flush=True)
