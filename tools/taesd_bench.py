"""Time the TAESD decoder (tools/; diagnostics): F frames per decode, CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_22009_b200 import vae as V  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 32
dec = V.TinyDecoder(seed=0, max_frames=F)
lat = torch.randn(F, 4, 64, 64, device="cuda")
out = torch.empty(F, 3, 512, 512, device="cuda")
for _ in range(3):
    dec.decode(lat, out)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    dec.decode(lat, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"taesd decode F={F}: {ms:.3f} ms  {F / ms * 1e3:.0f} frames/s  "
      f"{V.TinyDecoder.flops_per_frame() * F / ms / 1e9:.0f} TFLOP/s")
# per-layer split at the largest stage
H = 512
x = torch.zeros(F, H + 2, H + 2, 64, dtype=torch.bfloat16, device="cuda")
x[:, 1:-1, 1:-1] = torch.randn(F, H, H, 64, device="cuda").to(torch.bfloat16)
w = dec.conv_w[-1]
b = dec.conv_b[-1]
for epi in (V.EPI_NONE, V.EPI_RELU, V.EPI_RES_RELU):
    o = torch.zeros_like(x)
    for _ in range(2):
        V.conv3x3(x, w, b, epi, x, o)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        V.conv3x3(x, w, b, epi, x, o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    fl = 2.0 * F * H * H * 64 * 64 * 9
    by = F * (H + 2) ** 2 * 128 * (3 if epi == V.EPI_RES_RELU else 2)
    print(f"conv 512^2 epi={epi}: {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s  {by / ms / 1e6:.0f} GB/s (min traffic)")
