"""Standalone timing of the tcgen05 GEMM at DiT-S/2 shapes (diagnostics)."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_22009_b200 import _lib

M = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
st = torch.cuda.current_stream().cuda_stream
for (N, K, epi, name) in [(1536, 384, 2, "fc1 gelu"), (1536, 384, 1, "fc1 bf16"), (1536, 384, 0x102, "fc1 gelu nostore"),
                          (1536, 384, 0x101, "fc1 bf16 nostore"), (384 * 2, 1536, 1, "Kbig bf16 N768"),
                          (384 * 2, 1536, 0x101, "Kbig nostore")]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    b = torch.zeros(N, device="cuda")
    o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if (epi & 0xff) else torch.float32)
    for _ in range(3):
        _lib.call("sf_gemm_bf16", a.data_ptr(), w.data_ptr(), b.data_ptr(), o.data_ptr(), M, N, K, epi, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        _lib.call("sf_gemm_bf16", a.data_ptr(), w.data_ptr(), b.data_ptr(), o.data_ptr(), M, N, K, epi, st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:20s} M={M} N={N} K={K}: {ms*1e3:8.1f} us  {2*M*N*K/ms/1e9:7.1f} TFLOP/s")
