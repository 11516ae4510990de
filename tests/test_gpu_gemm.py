"""tcgen05 GEMM (sm_100a) against a torch fp32 reference of the same op."""

import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2511_22009_b200 import _lib as L
    return L


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 256, 384), (4096, 1536, 384),
                                   (1000, 384, 384), (2048, 1152, 1536), (300, 768, 256)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_matches_torch(M, N, K, epi):
    L = _lib()
    torch.manual_seed(M + N + K + epi)
    dev = "cuda"
    a = (torch.randn(M, K, device=dev) * 0.5).to(torch.bfloat16)
    w = (torch.randn(N, K, device=dev) * 0.05).to(torch.bfloat16)
    bias = torch.randn(N, device=dev, dtype=torch.float32) * 0.1
    out = torch.empty(M, N, device=dev, dtype=torch.float32 if epi == 0 else torch.bfloat16)
    L.call("sf_gemm_bf16", a.data_ptr(), w.data_ptr(), bias.data_ptr(), out.data_ptr(), M, N, K, epi,
           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = a.float() @ w.float().t() + bias
    if epi == 2:
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
    err = (out.float() - ref).abs().max().item()
    tol = 1e-3 if epi == 0 else 2e-2 * max(1.0, ref.abs().max().item())
    assert err <= tol, (M, N, K, epi, err)
