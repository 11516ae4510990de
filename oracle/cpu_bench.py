"""CPU baseline of the stream-batch hot path (TEST / BENCH INFRASTRUCTURE ONLY).

Times the oracle port (oracle/flowpipe_oracle.py's Euler step and queue +
oracle/dit_oracle.py's torch-fp32 DiT) on the host cores: one stream of the
bench workload (n slots at stages 0..n-1, steady state, one frame retires per
iteration).  The reference itself has no DiT and no GPU path, so
this port is the reference's CPU implementation of the path at the bench
shape ("kind": "port").  Used only by bench.py's cpu_baseline leg and
``--impl reference``.
"""

from __future__ import annotations

import os
import time

import numpy as np
import torch

from . import flowpipe_oracle as O
from .dit_oracle import dit_forward


class CpuStream:
    """One stream at steady state: n in-flight latents, newest first."""

    def __init__(self, params: dict, heads: int, n: int = 4, num_windows: int = 4, w: float = 1.0,
                 seed: int = 0, dim: int = 16384, embed_dim: int = 8):
        self.params, self.heads, self.n, self.w, self.dim = params, heads, n, w, dim
        self.sch = O.make_schedule(num_windows=num_windows, steps=n)
        self.seed = seed
        self.emb = O.conditioning_embedding(seed, embed_dim)
        self.next_id = n
        # generations n-1 .. 0 at stages 0 .. n-1 (batch order newest first)
        self.gens = list(range(n - 1, -1, -1))
        self.x = np.stack([O.generation_noise(seed, g, dim).astype(np.float32) for g in self.gens])

    def iteration(self) -> np.ndarray:
        """One stream-batch iteration: guided forward over n rows, Euler, retire
        the oldest, admit a fresh generation.  Returns the retired latent."""
        B = len(self.gens)
        ts = self.sch.grid[[self.n - 1 - i for i in range(B)]]
        xt = torch.from_numpy(self.x).view(B, 4, 64, 64)
        tt = torch.as_tensor(ts, dtype=torch.float64)
        ec = torch.as_tensor(np.tile(self.emb, (B, 1)))
        e = dit_forward(self.params, xt, tt, ec, self.heads).reshape(B, -1)
        if self.w != 1.0:
            eu = dit_forward(self.params, xt, tt, torch.zeros_like(ec), self.heads).reshape(B, -1)
            e = eu + self.w * (e - eu)
        x_new, _ = O.euler_step(e.numpy(), self.x, ts, self.sch)
        done = x_new[-1].copy()
        fresh = O.generation_noise(self.seed, self.next_id, self.dim).astype(np.float32)
        self.x = np.concatenate([fresh[None], x_new[:-1]])
        self.gens = [self.next_id] + self.gens[:-1]
        self.next_id += 1
        return done


def cpu_stream_throughput(params: dict, heads: int, iters: int = 2, warmup: int = 1, threads: int | None = None,
                          **kw) -> dict:
    """frames/s of one stream on `threads` host cores (one frame per iteration)."""
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    cs = CpuStream(params, heads, **kw)
    for _ in range(warmup):
        cs.iteration()
    times = []
    for _ in range(iters):
        t0 = time.perf_counter()
        cs.iteration()
        times.append(time.perf_counter() - t0)
    it = float(np.median(times))
    return {"frames_per_s": 1.0 / it, "iteration_s": times, "threads": threads,
            "p50_latency_ms": 1e3 * it * cs.n}
