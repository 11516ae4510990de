"""Standalone timing + accuracy of sf_attention at the bench shape (diagnostics):
rows x 6 heads x 1024 tokens x hd 64 (rows=128 = 32 streams x 4 slots)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_22009_b200 import _lib  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 128
H, T = 6, 1024
st = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda").manual_seed(0)
for scale in (1.0, 8.0):
    q = (torch.randn(rows, H, T, 64, device="cuda", generator=g) * scale / 8).to(torch.bfloat16)
    k = torch.randn(rows, H, T, 64, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(rows, H, T, 64, device="cuda", generator=g).to(torch.bfloat16)
    vt = v.transpose(-1, -2).contiguous().to(torch.float16)
    out = torch.empty(rows * T, H * 64, device="cuda", dtype=torch.bfloat16)
    call = lambda: _lib.call("sf_attention", q.data_ptr(), k.data_ptr(), vt.data_ptr(), out.data_ptr(), rows, H, T, st)
    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    fl = 4.0 * rows * H * T * T * 64
    n = min(rows, 4)
    ref = torch.nn.functional.scaled_dot_product_attention(q[:n].float(), k[:n].float(), v[:n].float(), scale=1.0)
    ref = ref.permute(0, 2, 1, 3).reshape(n * T, H * 64)
    err = (out[: n * T].float() - ref).abs().max().item()
    print(f"attention rows={rows} scale={scale}: {ms * 1e3:8.1f} us  {fl / ms / 1e9:7.1f} TFLOP/s  max|err|={err:.3e}")
