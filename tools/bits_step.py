"""Hash of the ring and frames after a few eager stream-batch steps: run under two builds
(SF_LIB_PATH=...) to show a kernel change is bit-identical end to end."""
import argparse
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22009_b200 as sf  # noqa: E402
from paper_2511_22009_b200.dit import DIT_S2, DIT_XL2  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--streams", type=int, default=32)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--xl", action="store_true")
ap.add_argument("--guidance", type=float, default=1.0)
a = ap.parse_args()
n = 4
cfgm = 2 if a.guidance != 1.0 else 1
model = sf.DiTVelocityModel(DIT_XL2 if a.xl else DIT_S2, seed=0, max_rows=cfgm * a.streams * n)
sched = sf.build_time_window_schedule(inference_steps=n)
conds = [sf.make_conditioning(np.random.default_rng([s, 5]).standard_normal(8), guidance_scale=a.guidance)
         for s in range(a.streams)]
sb = sf.StreamBatch(model, sched, n, num_streams=a.streams, cond=conds, seed=0, dtype=np.float32, noise="device",
                    use_graph=False)
h = hashlib.sha256()
for _ in range(a.steps):
    sb.launch()
    torch.cuda.synchronize()
    h.update(sb.x_ring.cpu().numpy().tobytes())
    h.update(sb.frames.cpu().numpy().tobytes())
print("bits", "xl" if a.xl else "s2", a.streams, a.guidance, h.hexdigest()[:16])
