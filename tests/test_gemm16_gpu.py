"""The training GEMM (csrc/ks_gemm16.cu, `ks_gemm_f16x3`) against fp64 torch:
every operand-major combination (K-major / MN-major A and B), ragged M, N, K
(TMA out-of-bounds fill, partial tiles), both tile widths, split-K shapes
(long reductions with few output tiles: the weight gradients) and beta = 1
accumulation.  Bar: fp32-grade -- |C - C64| <= 2e-5 x (|A| |B|) elementwise:
the F16X3 split is ~2^-22 per product, and fp32 accumulation over K up to
32,768 adds ~sqrt(K) 2^-24 (the order an fp32 SGEMM lands at; measured
worst cases here 5e-6 .. 8.5e-6)."""
import pytest
import torch

from tests.util import have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a GPU")]

SHAPES = [
    (60, 200, 1000),     # narrow M (slot rows), ragged N and K
    (130, 17, 70),       # tiny / ragged everything, 128-wide tiles
    (4096, 2048, 1024),  # decoder forward gates
    (4096, 1024, 2048),  # decoder dX
    (1024, 2048, 32768), # decoder dW: split-K
    (256, 1024, 28672),  # encoder dW: split-K, few tiles
]


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_f16x3_matches_fp64(shape, ta, tb):
    from paper_2404_10162_b200._cabi import gemm_f16x3
    M, N, K = shape
    g = torch.Generator(device="cpu").manual_seed(M * 31 + N * 7 + K + 2 * ta + tb)
    A = torch.randn((K, M) if ta else (M, K), generator=g, dtype=torch.float64)
    B = torch.randn((N, K) if tb else (K, N), generator=g, dtype=torch.float64)
    A[0, 0] *= 300.0  # a large entry: the per-operand scale must keep the rest exact
    opA = A.T if ta else A
    opB = B.T if tb else B
    ref = opA @ opB
    bound = opA.abs() @ opB.abs()
    C = gemm_f16x3(A.float().cuda(), B.float().cuda(), ta=ta, tb=tb)
    err = ((C.double().cpu() - ref).abs() / (bound + 1e-30)).max().item()
    assert err < 2e-5, err


def test_gemm_f16x3_beta_one_accumulates():
    from paper_2404_10162_b200._cabi import gemm_f16x3
    M, N, K = 512, 768, 4096
    g = torch.Generator(device="cpu").manual_seed(5)
    A = torch.randn((M, K), generator=g, dtype=torch.float64)
    B = torch.randn((K, N), generator=g, dtype=torch.float64)
    C0 = torch.randn((M, N), generator=g, dtype=torch.float64)
    C = gemm_f16x3(A.float().cuda(), B.float().cuda(), C=C0.float().cuda(), beta=1.0)
    ref = A @ B + C0
    bound = A.abs() @ B.abs() + C0.abs()
    assert ((C.double().cpu() - ref).abs() / bound).max().item() < 2e-5
