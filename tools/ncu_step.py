"""Minimal driver for ncu captures: build the bench workload and run a few
eager (non-graph) stream-batch steps so every kernel launch is visible."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22009_b200 as sf  # noqa: E402
from paper_2511_22009_b200.dit import DIT_S2  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--streams", type=int, default=32)
ap.add_argument("--n", type=int, default=4)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--graph", action="store_true")
a = ap.parse_args()
model = sf.DiTVelocityModel(DIT_S2, seed=0, max_rows=a.streams * a.n)
sched = sf.build_time_window_schedule(inference_steps=a.n)
conds = [sf.make_conditioning(np.random.default_rng([s, 2**32 - 1]).standard_normal(8)) for s in range(a.streams)]
sb = sf.StreamBatch(model, sched, a.n, num_streams=a.streams, cond=conds, seed=0, dtype=np.float32,
                    noise="device", use_graph=a.graph)
for _ in range(a.steps):
    sb.launch()
torch.cuda.synchronize()
print("done", sb.j)
