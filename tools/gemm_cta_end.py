"""Per-CTA end times of the DiT-S/2 QKV GEMM (pair tiles, weight slice resident; library built with
-DSF_GEMM_TRACE=1): are the pairs that own V column slices (transposed V^T epilogue) the last ones?"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_22009_b200 import _lib  # noqa: E402

M, D, T, H = 131072, 384, 1024, 6
st = torch.cuda.current_stream().cuda_stream
bf = lambda t: t.to(torch.bfloat16)  # noqa: E731
a = bf(torch.randn(M, D, device="cuda"))
w = bf(torch.randn(3 * D, D, device="cuda") * 0.05)
b = torch.zeros(3 * D, device="cuda")
q = torch.empty(M // T, H, T, 64, device="cuda", dtype=torch.bfloat16)
k = torch.empty_like(q)
vt = torch.empty(M // T, H, 64, T, device="cuda", dtype=torch.float16)
lib = _lib.load()
for rep in range(3):
    _lib.call("sf_gemm_qkv", a.data_ptr(), w.data_ptr(), b.data_ptr(), q.data_ptr(), k.data_ptr(), vt.data_ptr(), M,
              H, T, 0.125, st)
    torch.cuda.synchronize()
    ends = (ctypes.c_ulonglong * 1024)()
    lib.sf_gemm_cta_end_read(ends)
    e = np.array(ends[:144], dtype=np.float64)
    e -= e.min()
    pairs = e.reshape(72, 2).max(axis=1) / 1e3  # us after the first CTA finished
    by_slice = [pairs[s::6] for s in range(6)]
    print(f"rep {rep}: per column slice (Q0 Q1 K0 K1 V0 V1) mean / max end (us after first): "
          + "  ".join(f"{x.mean():.1f}/{x.max():.1f}" for x in by_slice))
