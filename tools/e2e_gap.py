"""Where does bench's e2e line lose to its device-resident value?  Times the same S=32 DiT-S/2
stream batch four ways (CUDA events, 40 steps after warm-up): noise='device' launch(),
noise='host' launch() (device-resident noise buffer), launch_host_io (side-stream copies), and
noise='device' again (clock drift check)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22009_b200 as sf  # noqa: E402
from paper_2511_22009_b200.dit import DIT_S2  # noqa: E402

S, n, K = 32, 4, 40
model = sf.DiTVelocityModel(DIT_S2, seed=0, max_rows=S * n)
sched = sf.build_time_window_schedule(num_windows=4, inference_steps=n)
conds = [sf.make_conditioning(np.random.default_rng([s, 7]).standard_normal(8)) for s in range(S)]


def run(noise, io):
    sb = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=1000, dtype=np.float32, noise=noise)
    pool = [torch.randn(S, model.dim).pin_memory() for _ in range(2)]
    dst = torch.empty(S, model.dim).pin_memory()
    step = (lambda i: sb.launch_host_io(pool[i % 2], dst)) if io else (lambda i: sb.launch())
    for i in range(6):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(K):
        step(i)
    if io:
        sb.io_join()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    return ms, S / ms * 1e3


for name, noise, io in (("device", "device", False), ("host-noise launch", "host", False),
                        ("launch_host_io", "host", True), ("device again", "device", False)):
    ms, fps = run(noise, io)
    print(f"{name:20s} {ms:7.3f} ms/step  {fps:7.1f} frames/s")
