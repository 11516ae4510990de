"""HBM write-only / read-only / copy bandwidth (torch kernels, CUDA events)."""
import torch
n = 400 * 1024 * 1024 // 2
x = torch.empty(n, dtype=torch.bfloat16, device="cuda")
y = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
def t(fn, bytes_, name):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:12s} {bytes_ / ms / 1e6:8.1f} GB/s ({ms*1e3:.1f} us for {bytes_/1e6:.0f} MB)")
t(lambda: x.fill_(1.0), 2 * n, "write-only")
t(lambda: y.sum(), 2 * n, "read-only")
t(lambda: x.copy_(y), 4 * n, "copy r+w")
