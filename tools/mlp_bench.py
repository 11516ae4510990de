"""Fused MLP block (sf_mlp_fused) vs the unfused fc1 GELU GEMM + fc2 RES_LN GEMM at the
bench shape (M = 131072 tokens); diagnostics."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_22009_b200 import _lib  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
T, N, F = 1024, 384, 1536
st = torch.cuda.current_stream().cuda_stream
bf = lambda t: t.to(torch.bfloat16)
x = bf(torch.randn(M, N, device="cuda"))
w1 = bf(torch.randn(F, N, device="cuda") * 0.05)
b1 = torch.zeros(F, device="cuda")
w2 = bf(torch.randn(N, F, device="cuda") * 0.03)
b2 = torch.zeros(N, device="cuda")
xres = bf(torch.randn(M, N, device="cuda"))
xmod = x.clone()
vecs = torch.randn(M // T, 4 * N, device="cuda") * 0.1
h = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)


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
    return e0.elapsed_time(e1) / n * 1e3


def fused():
    _lib.call("sf_mlp_fused", xmod.data_ptr(), w1.data_ptr(), w2.data_ptr(), b1.data_ptr(), b2.data_ptr(),
              xres.data_ptr(), xmod.data_ptr(), vecs.data_ptr(), vecs[:, N:].data_ptr(), vecs[:, 2 * N:].data_ptr(),
              4 * N, 1e-6, M, T, st)


def unfused():
    _lib.call("sf_gemm_bf16", x.data_ptr(), w1.data_ptr(), b1.data_ptr(), h.data_ptr(), M, F, N, 2, st)
    _lib.call("sf_gemm_res_ln", h.data_ptr(), w2.data_ptr(), b2.data_ptr(), xres.data_ptr(), xmod.data_ptr(),
              vecs.data_ptr(), vecs[:, N:].data_ptr(), vecs[:, 2 * N:].data_ptr(), 4 * N, M, N, F, T, 1e-6, st)


fl = 2 * 2.0 * M * N * F
for name, fn in (("fused", fused), ("unfused", unfused)):
    us = timeit(fn)
    print(f"mlp {name:8s}: {us:8.1f} us  {fl / us / 1e6:7.1f} TFLOP/s")

# post-attention block tail (projection + MLP) vs the projection GEMM + fused MLP
attn = bf(torch.randn(M, N, device="cuda"))
wp = bf(torch.randn(N, N, device="cuda") * 0.05)
bp = torch.zeros(N, device="cuda")
v8 = torch.randn(M // T, 8 * N, device="cuda") * 0.1


def tail():
    _lib.call("sf_block_tail", attn.data_ptr(), wp.data_ptr(), bp.data_ptr(), w1.data_ptr(), w2.data_ptr(),
              b1.data_ptr(), b2.data_ptr(), xres.data_ptr(), xmod.data_ptr(), v8.data_ptr(), v8[:, N:].data_ptr(),
              v8[:, 2 * N:].data_ptr(), v8[:, 3 * N:].data_ptr(), v8[:, 4 * N:].data_ptr(), v8[:, 5 * N:].data_ptr(),
              8 * N, 1e-6, M, T, st)


def two():
    _lib.call("sf_gemm_res_ln", attn.data_ptr(), wp.data_ptr(), bp.data_ptr(), xres.data_ptr(), xmod.data_ptr(),
              v8.data_ptr(), v8[:, N:].data_ptr(), v8[:, 2 * N:].data_ptr(), 8 * N, M, N, N, T, 1e-6, st)
    fused()


fl2 = fl + 2.0 * M * N * N
for name, fn in (("tail", tail), ("proj+mlp", two)):
    us = timeit(fn)
    print(f"block {name:8s}: {us:8.1f} us  {fl2 / us / 1e6:7.1f} TFLOP/s")
