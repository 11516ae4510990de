"""Standalone block-tail launches at the bench shape (M = 128 latents x 1024 tokens), for ncu
and quick timing: python tools/tail_bench.py [--iters N]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_22009_b200 import _lib  # noqa: E402

iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 10
T, N, F = 1024, 384, 1536
slots = int(os.environ.get("SLOTS", "128"))
M = slots * T
g = torch.Generator(device="cuda").manual_seed(0)
bf = lambda x: x.to(torch.bfloat16)
attn = bf(torch.randn(M, N, device="cuda", generator=g))
wp = bf(torch.randn(N, N, device="cuda", generator=g) * 0.05)
w1 = bf(torch.randn(F, N, device="cuda", generator=g) * 0.05)
w2 = bf(torch.randn(N, F, device="cuda", generator=g) * 0.03)
bp, b1, b2 = (torch.zeros(n, device="cuda") for n in (N, F, N))
xres = bf(torch.randn(M, N, device="cuda", generator=g))
xmod = torch.empty_like(xres)
vecs = torch.randn(slots, 8 * N, device="cuda", generator=g) * 0.1
P = lambda t: t.data_ptr()
st = torch.cuda.current_stream().cuda_stream
args = [P(attn), P(wp), P(bp), P(w1), P(w2), P(b1), P(b2), P(xres), P(xmod)] + \
       [P(vecs[:, i * N:]) for i in range(6)] + [8 * N, 1e-6, M, T, st]
for _ in range(2):
    _lib.call("sf_block_tail", *args)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(iters):
    _lib.call("sf_block_tail", *args)
ev[1].record()
torch.cuda.synchronize()
print(f"block tail: {ev[0].elapsed_time(ev[1]) / iters * 1e3:.1f} us per launch at M={M}")
