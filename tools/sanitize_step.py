"""Driver for compute-sanitizer (racecheck / synccheck / memcheck) runs of the hot path:
the mock stream step and the DiT-S/2 stream step, eager launches (every kernel visible),
at 40 latent rows (320 row tiles: the persistent kernels walk 2-3 tiles per CTA, so the
cross-tile pipeline phases run under the checker).  Usage:
    compute-sanitizer --tool racecheck python tools/sanitize_step.py [--rows-streams S]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22009_b200 as sf  # noqa: E402
from paper_2511_22009_b200.dit import DIT_S2, DIT_XL2  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--streams", type=int, default=10)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--guidance", type=float, default=1.0)
ap.add_argument("--xl", action="store_true", help="DiT-XL/2 stream step instead (pair-tile GEMMs, head dim 72)")
a = ap.parse_args()
n = 4
sched = sf.build_time_window_schedule(inference_steps=n)
mock = sf.SeededMockModel(dim=4096, seed=1)
cond = sf.make_conditioning(np.ones(8), guidance_scale=a.guidance)
res, _ = sf.run_stream(3, n, mock, cond, 5, sched)
model = sf.DiTVelocityModel(DIT_XL2 if a.xl else DIT_S2, seed=0, max_rows=2 * a.streams * n)
conds = [sf.make_conditioning(np.random.default_rng([s, 7]).standard_normal(8), guidance_scale=a.guidance)
         for s in range(a.streams)]
sb = sf.StreamBatch(model, sched, n, num_streams=a.streams, cond=conds, seed=0, dtype=np.float32, noise="device",
                    use_graph=False)
for _ in range(a.steps):
    sb.launch()
torch.cuda.synchronize()
assert torch.isfinite(sb.x_ring).all()
print("sanitize_step done", len(res), sb.j)
