import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2511_22009_b200 import _lib
H, T = 6, 1024
st = torch.cuda.current_stream().cuda_stream
for rows in (1, 8):
  for scale in (1.0, 2.0, 3.0, 4.0, 8.0):
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.randn(rows, H, T, 64, device="cuda", generator=g) * scale / 8).to(torch.bfloat16)
    k = torch.randn(rows, H, T, 64, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(rows, H, T, 64, device="cuda", generator=g).to(torch.bfloat16)
    vt = v.transpose(-1, -2).contiguous().to(torch.float16)
    out = torch.zeros(rows * T, H * 64, device="cuda", dtype=torch.bfloat16)
    _lib.call("sf_attention", q.data_ptr(), k.data_ptr(), vt.data_ptr(), out.data_ptr(), rows, H, T, st)
    torch.cuda.synchronize()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float(), scale=1.0)
    ref = ref.permute(0, 2, 1, 3).reshape(rows * T, H * 64)
    e = (out.float() - ref).abs().view(rows, T, H, 64).amax(-1)  # rows, T, H
    bad = (e > 0.05)
    print(f"rows={rows} scale={scale} maxerr={e.max().item():.3e} bad={bad.sum().item()} of {bad.numel()}")
    if bad.any():
        idx = bad.nonzero()[:8].tolist(); print("  first bad (row,q,head):", idx)
        qs = bad.any(0).any(1).nonzero().flatten()
        print("  bad q range", qs.min().item(), qs.max().item(), "count", qs.numel(), "q%128 hist", torch.bincount(qs % 128, minlength=128)[:8].tolist())
