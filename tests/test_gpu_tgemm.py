"""GPU parity of the tcgen05 bf16 GEMM building block (C-ABI dsmpnn_gemm_bf16)
against a plain fp64 product of the same bf16 inputs."""
import numpy as np
import pytest
import torch

from gpu_util import cuda, nerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2402_15106_b200 import build
    build.build()
    from paper_2402_15106_b200 import _lib
    return _lib


SHAPES = [(128, 64, 64), (200, 16, 104), (256, 32, 128), (300, 64, 520), (128, 128, 64), (384, 256, 256),
          (1000, 256, 16512), (4096, 64, 16512), (77, 48, 64)]


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_bf16(L, M, N, K, a_mn, b_mn):
    if b_mn and N > 64 and N % 64:
        pytest.skip("N-major B with N > 64 needs N % 64 == 0")
    if (a_mn and M % 8) or (b_mn and N % 8) or K % 8:
        pytest.skip("16-byte row alignment")
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = torch.randn(K, N, generator=g).to(torch.bfloat16)
    ref = A.double() @ B.double()
    Ad = (A.t().contiguous() if a_mn else A).to(cuda())
    Bd = (B if b_mn else B.t().contiguous()).to(cuda())
    C = torch.full((M, N), float("nan"), device=cuda())
    L.gemm_bf16(Ad, Bd, C, a_mn_major=a_mn, b_mn_major=b_mn, M=M, N=N, K=K)
    torch.cuda.synchronize()
    # fp32 tensor-core accumulation over K terms: allow ~1e-6 * sqrt(K)
    assert nerr(C.cpu().numpy(), ref.numpy()) < 2e-6 * max(8.0, K ** 0.5)


def test_gemm_bf16_splitk_accumulate(L):
    M, N, K = 256, 256, 8192
    g = torch.Generator().manual_seed(5)
    A = torch.randn(K, M, generator=g).to(torch.bfloat16)   # stored [K][M]: M-major A
    B = torch.randn(K, N, generator=g).to(torch.bfloat16)   # stored [K][N]: N-major B
    ref = A.double().t() @ B.double()
    C0 = torch.randn(M, N, generator=g)
    C = C0.clone().to(cuda())
    part = torch.empty(8 * M * N, device=cuda())
    L.gemm_bf16(A.to(cuda()), B.to(cuda()), C, a_mn_major=True, b_mn_major=True, splits=8, partial=part,
                accumulate=True, M=M, N=N, K=K)
    torch.cuda.synchronize()
    assert nerr(C.cpu().numpy(), (ref + C0.double()).numpy()) < 1e-5
