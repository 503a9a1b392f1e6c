"""tcgen05 3xTF32 GEMM (steps a2/a4/a5) in isolation, through the C-ABI debug entry.

Reference: plain float64 matmul of the same float32 inputs.  Tolerance: the
3xTF32 scheme keeps ~fp32 accuracy; we require max|C - C_ref| <= 1e-5 * (|A||B| row/col
scale) and check that 1xTF32 is measurably worse (5e-4 vs 3.7e-7)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2306_06528_b200 import push  # noqa: E402


def _mk(batch, M, N, K, a_mn, b_mn, seed):
    g = torch.Generator().manual_seed(seed)
    A = torch.randn(batch, M, K, generator=g, dtype=torch.float64)
    B = torch.randn(batch, K, N, generator=g, dtype=torch.float64)
    A32, B32 = A.float(), B.float()
    ref = torch.bmm(A32.double(), B32.double())
    Ad = (A32.transpose(1, 2) if a_mn else A32).contiguous().cuda()   # a_mn: [K][M]
    Bd = (B32 if b_mn else B32.transpose(1, 2)).contiguous().cuda()   # b_mn: [K][N]; else [N][K]
    scale = torch.bmm(A32.double().abs(), B32.double().abs())
    return Ad, Bd, ref, scale


@pytest.mark.parametrize("b_split", [0, 1])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 64, 96), (96, 32, 32), (300, 256, 128), (1, 32, 4),
                                   (640, 128, 1000), (512, 512, 256), (96, 256, 40), (1000, 768, 512)])
def test_gemm_3xtf32_matches_fp64(a_mn, b_mn, b_split, M, N, K):
    if a_mn and M % 32:
        pytest.skip("MN-major A needs M % 32 == 0")
    batch = 3
    Ad, Bd, ref, scale = _mk(batch, M, N, K, a_mn, b_mn, 1 + M + N + K)
    C = push.gemm3xtf32(Ad, Bd, bool(a_mn), bool(b_mn), M, N, K, b_split=bool(b_split)).double().cpu()
    err = ((C - ref).abs() / scale.clamp_min(1e-30)).max().item()
    assert err < 2e-6, err


def test_gemm_long_k_split_precision():
    # K = 4096: the weight-gradient shape (K = batch); 3xTF32 must beat 1xTF32 by >= 100x
    M, N, K = 128, 128, 4096
    Ad, Bd, ref, scale = _mk(2, M, N, K, 1, 1, 7)
    C3 = push.gemm3xtf32(Ad, Bd, True, True, M, N, K, passes=3, b_split=True).double().cpu()
    C1 = push.gemm3xtf32(Ad, Bd, True, True, M, N, K, passes=1, b_split=True).double().cpu()
    e3 = ((C3 - ref).abs().max() / ref.abs().max()).item()
    e1 = ((C1 - ref).abs().max() / ref.abs().max()).item()
    assert e3 < 1e-5, e3
    assert e1 > 100 * e3, (e1, e3)
