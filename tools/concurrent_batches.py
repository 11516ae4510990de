"""Experiment: the 32-stream workload as ONE S=32 batch vs TWO S=16 batches (two model handles,
two CUDA streams, graph replays interleaved) -- can a second batch fill the first one's kernel
tails / prologues?  CUDA events on a joined timeline, 30 steps after 6 warm-up, interleaved reps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22009_b200 as sf  # noqa: E402
from paper_2511_22009_b200.dit import DIT_S2  # noqa: E402

n, K = 4, 30
sched = sf.build_time_window_schedule(inference_steps=n)


def batch(model, S, s0):
    conds = [sf.make_conditioning(np.random.default_rng([s0 + s, 7]).standard_normal(8)) for s in range(S)]
    return sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=s0, dtype=np.float32, noise="device")


m32 = sf.DiTVelocityModel(DIT_S2, seed=0, max_rows=32 * n)
one = batch(m32, 32, 0)
ma = sf.DiTVelocityModel(DIT_S2, seed=0, max_rows=16 * n)
mb = sf.DiTVelocityModel(DIT_S2, seed=0, max_rows=16 * n)
half_a, half_b = batch(ma, 16, 0), batch(mb, 16, 16)
sa, sb_ = torch.cuda.Stream(), torch.cuda.Stream()


def run_one():
    one.launch()


def run_two():
    with torch.cuda.stream(sa):
        half_a.launch()
    with torch.cuda.stream(sb_):
        half_b.launch()


def timed(fn, two):
    for _ in range(6):
        fn()
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    if two:
        sa.wait_stream(cur)
        sb_.wait_stream(cur)
    for _ in range(K):
        fn()
    if two:
        cur.wait_stream(sa)
        cur.wait_stream(sb_)
    b.record(cur)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


for rep in range(3):
    t1 = timed(run_one, False)
    t2 = timed(run_two, True)
    print(f"rep {rep}: one S=32 batch {t1:.3f} ms/step ({32e3 / t1:.1f} frames/s); "
          f"two S=16 batches concurrently {t2:.3f} ms/step ({32e3 / t2:.1f} frames/s)")
