"""Diagnostics: DiT-XL/2 device forward vs fp32 reference, next to a torch-bf16 autocast reference."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.dit_oracle import dit_forward, params_to
from paper_2511_22009_b200.dit import DIT_XL2, DIT_S2, DeviceDiT, init_dit_params
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
for cfg, heads in ((DIT_S2, 6), (DIT_XL2, 16)):
    params = init_dit_params(cfg, seed=5, bias_std=0.02)
    dit = DeviceDiT(params, cfg, max_rows=4)
    g = torch.Generator().manual_seed(1)
    x = torch.randn(2, 4, 64, 64, generator=g)
    t = torch.tensor([0.0, 0.5], dtype=torch.float64)
    e = torch.randn(2, 8, generator=g, dtype=torch.float64)
    pc = params_to(params, "cuda")
    want = dit_forward(pc, x.cuda(), t.cuda(), e.cuda(), heads=heads)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        wb = dit_forward(pc, x.cuda(), t.cuda(), e.cuda(), heads=heads).float()
    got = dit.forward(x.cuda(), t.cuda(), e.cuda()).view(2, 4, 64, 64)
    s = want.abs().max().item()
    for name, v in (("device", got), ("torch-bf16", wb)):
        d = (v - want).abs()
        print(f"{cfg.hidden} {name:10s} max {d.max().item()/s:.4f} mean {d.mean().item()/s:.5f}")
