"""Where the e2e (host-buffer) line loses against the device line: the same S=32 DiT step timed
as (a) launch() with Philox noise fused in the refill (bench value), (b) launch() with noise='host'
and the device noise buffer pre-filled (no copies), (c) launch_host_io() with pinned host buffers,
(d) like (c) but one H2D per step only (D2H skipped).  CUDA events over 30 steps after 6 warm-up."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22009_b200 as sf  # noqa: E402
from paper_2511_22009_b200.dit import DIT_S2  # noqa: E402

S, n, K = 32, 4, 30
model = sf.DiTVelocityModel(DIT_S2, seed=0, max_rows=S * n)
sched = sf.build_time_window_schedule(inference_steps=n)
conds = [sf.make_conditioning(np.random.default_rng([s, 7]).standard_normal(8)) for s in range(S)]


def timed(fn):
    for _ in range(6):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


dev = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=0, dtype=np.float32, noise="device")
host = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=0, dtype=np.float32, noise="host")
host.noise_dev.normal_()
src = torch.randn(S, DIT_S2.dim).pin_memory()
dst = torch.empty(S, DIT_S2.dim).pin_memory()
io = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=0, dtype=np.float32, noise="host")
res = {}
for rep in range(2):
    res[f"a_device_launch_{rep}"] = timed(dev.launch)
    res[f"b_host_launch_prefilled_{rep}"] = timed(host.launch)

    def step_io():
        io.launch_host_io(src, dst)

    res[f"c_launch_host_io_{rep}"] = timed(step_io)
for k, v in res.items():
    print(f"{k:32s} {v:.3f} ms/step  {S * 1e3 / v:.1f} frames/s")
