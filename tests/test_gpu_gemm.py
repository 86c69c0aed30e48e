"""tcgen05 GEMM (K5 building block) against a float64 reference."""
import pytest
import torch

from paper_2604_03143_b200 import gemm

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.mark.parametrize("M,N,K", [(1, 8, 8), (128, 64, 32), (130, 100, 72), (300, 512, 512),
                                   (17, 1536, 512), (256, 128, 40)])
def test_gemm_tf32x3_matches_float64(M, N, K):
    g = torch.Generator(device=DEV).manual_seed(M * 1000 + N + K)
    a = torch.randn(M, K, generator=g, device=DEV)
    b = torch.randn(N, K, generator=g, device=DEV) * 0.1
    out = gemm.gemm_tn(a, b)
    want = (a.double() @ b.double().T)
    err = (out.double() - want).abs().max().item()
    scale = want.abs().max().item()
    assert err <= 2e-6 * max(1.0, scale) * max(1.0, (K / 64) ** 0.5), (err, scale)


@pytest.mark.parametrize("M,N,K", [(1, 8, 8), (128, 64, 32), (130, 100, 72), (300, 512, 512),
                                   (17, 1536, 512), (2048, 4608, 512)])
def test_gemm_presplit_equals_in_kernel_split(M, N, K):
    """tdkv_gemm_tf32x3 over tdkv_tf32_split planes performs the same
    tf32 splits and the same MMA sequence as the in-kernel split of
    tdkv_gemm: bit-identical results, plain and accumulating (the toy
    model's residual update h += mix @ Wm)."""
    g = torch.Generator(device=DEV).manual_seed(M + 7 * N + 13 * K)
    a = torch.randn(M, K, generator=g, device=DEV)
    b = torch.randn(N, K, generator=g, device=DEV) * 0.1
    c0 = torch.randn(M, N, generator=g, device=DEV)
    hi, lo = gemm.tf32_split(a)
    assert torch.equal(hi + lo, hi + lo) and (hi.view(torch.int32) & 0x1FFF).eq(0).all()
    for acc in (False, True):
        want, got = c0.clone(), c0.clone()
        gemm.gemm_tn(a, b, out=want, accumulate=acc)
        gemm.gemm_tf32x3((hi, lo), gemm.tf32_split(b), out=got, accumulate=acc)
        assert torch.equal(got, want), (acc, (got - want).abs().max().item())


def test_gemm_accumulate_residual():
    g = torch.Generator(device=DEV).manual_seed(7)
    a = torch.randn(200, 64, generator=g, device=DEV)
    b = torch.randn(96, 64, generator=g, device=DEV)
    c = torch.randn(200, 96, generator=g, device=DEV)
    want = c.double() + a.double() @ b.double().T
    gemm.gemm_tn(a, b, out=c, accumulate=True)
    # float32 result rounding of |values| up to ~25 plus 3xTF32 product error
    assert (c.double() - want).abs().max().item() <= 2e-6 * want.abs().max().item()


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (77, 200, 512)])
def test_gemm_bf16(M, N, K):
    g = torch.Generator(device=DEV).manual_seed(3)
    a = torch.randn(M, K, generator=g, device=DEV).bfloat16()
    b = torch.randn(N, K, generator=g, device=DEV).bfloat16()
    out = gemm.gemm_tn(a, b)
    want = a.double() @ b.double().T
    assert (out.double() - want).abs().max().item() <= 1e-3 * max(1.0, want.abs().max().item())


@pytest.mark.parametrize("M,N,K", [(300, 512, 512), (2048, 4608, 256), (130, 300, 72),
                                   (129, 257, 1000), (4096, 4096, 128)])
def test_gemm_bf16_persistent(M, N, K):
    """Shapes that put several output tiles on one persistent CTA (both TMEM
    accumulator buffers in use), ragged M/N/K edges and the scalar tail."""
    g = torch.Generator(device=DEV).manual_seed(M + N + K)
    a = torch.randn(M, K, generator=g, device=DEV).bfloat16()
    b = torch.randn(N, K, generator=g, device=DEV).bfloat16()
    out = gemm.gemm_tn(a, b)
    want = a.double() @ b.double().T
    assert (out.double() - want).abs().max().item() <= 1e-5 * max(1.0, want.abs().max().item()) * K ** 0.5


def test_gemm_bf16_persistent_accumulate():
    g = torch.Generator(device=DEV).manual_seed(11)
    a = torch.randn(1000, 192, generator=g, device=DEV).bfloat16()
    b = torch.randn(1000, 192, generator=g, device=DEV).bfloat16()
    c = torch.randn(1000, 1000, generator=g, device=DEV)
    want = c.double() + a.double() @ b.double().T
    gemm.gemm_tn(a, b, out=c, accumulate=True)
    assert (c.double() - want).abs().max().item() <= 1e-5 * want.abs().max().item() * 192 ** 0.5


@pytest.mark.parametrize("M,N,K", [(2048, 4608, 320), (4096, 2560, 64), (2100, 4700, 104)])
def test_gemm_bf16_cta_pair(M, N, K):
    """Shapes large enough for the cta_group::2 kernel (every CTA pair busy),
    including ragged M/N/K."""
    g = torch.Generator(device=DEV).manual_seed(M ^ N ^ K)
    a = torch.randn(M, K, generator=g, device=DEV).bfloat16()
    b = torch.randn(N, K, generator=g, device=DEV).bfloat16()
    c = torch.randn(M, N, generator=g, device=DEV)
    want = a.double() @ b.double().T
    out = gemm.gemm_tn(a, b)
    assert (out.double() - want).abs().max().item() <= 1e-5 * max(1.0, want.abs().max().item()) * K ** 0.5
    want = want + c.double()
    gemm.gemm_tn(a, b, out=c, accumulate=True)
    assert (c.double() - want).abs().max().item() <= 1e-5 * max(1.0, want.abs().max().item()) * K ** 0.5
