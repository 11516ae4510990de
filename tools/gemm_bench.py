"""Standalone timing of the layer GEMMs at the bench shape (M = 131072 tokens):
QKV (+head-major scatter), proj (+gated residual + LN + modulate), fc1 (+GELU),
fc2 (+gated residual + LN + modulate).  Diagnostics only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_22009_b200 import _lib  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 131072
T, H, D = 1024, 6, 384
st = torch.cuda.current_stream().cuda_stream
bf = lambda t: t.to(torch.bfloat16)
dev = "cuda"


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


a = bf(torch.randn(M, D, device=dev))
h = bf(torch.randn(M, 4 * D, device=dev))
rows = M // T
# QKV
w = bf(torch.randn(3 * D, D, device=dev) * 0.05)
b = torch.zeros(3 * D, device=dev)
q = torch.empty(rows, H, T, 64, device=dev, dtype=torch.bfloat16)
k = torch.empty_like(q)
vt = torch.empty(rows, H, 64, T, device=dev, dtype=torch.float16)
ms = timeit(lambda: _lib.call("sf_gemm_qkv", a.data_ptr(), w.data_ptr(), b.data_ptr(), q.data_ptr(), k.data_ptr(),
                              vt.data_ptr(), M, H, T, 0.125, st))
print(f"qkv   N={3*D} K={D}: {ms*1e3:7.1f} us {2*M*3*D*D/ms/1e9:7.1f} TFLOP/s")
# fc1
w1 = bf(torch.randn(4 * D, D, device=dev) * 0.05)
b1 = torch.zeros(4 * D, device=dev)
o1 = torch.empty(M, 4 * D, device=dev, dtype=torch.bfloat16)
ms = timeit(lambda: _lib.call("sf_gemm_bf16", a.data_ptr(), w1.data_ptr(), b1.data_ptr(), o1.data_ptr(), M, 4 * D, D,
                              2, st))
print(f"fc1   N={4*D} K={D}: {ms*1e3:7.1f} us {2*M*4*D*D/ms/1e9:7.1f} TFLOP/s")
# proj / fc2 (res + LN)
for name, A, K in (("proj", a, D), ("fc2", h, 4 * D)):
    w2 = bf(torch.randn(D, K, device=dev) * 0.05)
    b2 = torch.zeros(D, device=dev)
    xres = bf(torch.randn(M, D, device=dev))
    xmod = torch.empty(M, D, device=dev, dtype=torch.bfloat16)
    vec = torch.randn(rows, 3 * D, device=dev) * 0.1
    ms = timeit(lambda: _lib.call("sf_gemm_res_ln", A.data_ptr(), w2.data_ptr(), b2.data_ptr(), xres.data_ptr(),
                                  xmod.data_ptr(), vec.data_ptr(), vec[:, D:].data_ptr(), vec[:, 2 * D:].data_ptr(),
                                  3 * D, M, D, K, T, 1e-6, st))
    print(f"{name:5s} N={D} K={K}: {ms*1e3:7.1f} us {2*M*D*K/ms/1e9:7.1f} TFLOP/s")
# diagnostics: fc1-shaped GEMM with the epilogue stores skipped (0x100) / the epilogue skipped (0x200)
for flag, name in ((0x102, "fc1 gelu nostore"), (0x101, "fc1 bf16 nostore"), (0x201, "fc1 mainloop only")):
    ms = timeit(lambda: _lib.call("sf_gemm_bf16", a.data_ptr(), w1.data_ptr(), b1.data_ptr(), o1.data_ptr(), M, 4 * D,
                                  D, flag, st))
    print(f"{name:18s}: {ms*1e3:7.1f} us {2*M*4*D*D/ms/1e9:7.1f} TFLOP/s")
for name, A, K in (("proj", a, D), ("fc2", h, 4 * D)):
    w2 = bf(torch.randn(D, K, device=dev) * 0.05)
    b2 = torch.zeros(D, device=dev)
    xres = bf(torch.randn(M, D, device=dev))
    xmod = torch.empty(M, D, device=dev, dtype=torch.bfloat16)
    vec = torch.randn(rows, 3 * D, device=dev) * 0.1
    ms = timeit(lambda: _lib.call("sf_gemm_res_ln", A.data_ptr(), w2.data_ptr(), b2.data_ptr(), xres.data_ptr(),
                                  xmod.data_ptr(), vec.data_ptr(), vec[:, D:].data_ptr(), vec[:, 2 * D:].data_ptr(),
                                  3 * D, M, D, K, T, 1e-6, st))
    print(f"{name:5s} res+LN N={D} K={K}: {ms*1e3:7.1f} us {2*M*D*K/ms/1e9:7.1f} TFLOP/s")
