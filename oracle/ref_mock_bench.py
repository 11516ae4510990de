"""Times the UNMODIFIED reference package's own CPU path (BENCH INFRASTRUCTURE ONLY).

BASELINE.md section 3 "Oracle A": ``flowpipe.run_stream`` with
``SeededMockModel(dim=16384)`` -- the reference's config[0] "small velocity model"
(models.py:199-241) through its own stream loop (pipeline.py:139-220) -- in fp64 and
fp32, on one process (per-stream latency) and on ``os.cpu_count()`` processes, one
independent stream each (aggregate frames/s; numpy elementwise work is single-threaded).

The reference is imported from ``baseline/_ref`` (``pip install --no-index --target
baseline/_ref /root/reference``, recorded in DESIGN.md); when that install is absent the
oracle restatement (oracle/flowpipe_oracle.py) is timed instead and the result says
``kind: "port"``.  Used only by bench.py's cpu_baseline leg and ``--impl reference``.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF, "flowpipe"))


def _one_stream(args):
    """m generations of one stream through flowpipe.run_stream; returns (seconds, frames,
    per-frame latency ms from the on_iteration stamps)."""
    m, n, dim, seed, dtype_name, use_ref = args
    dtype = np.float64 if dtype_name == "f64" else np.float32
    if use_ref:
        if REF not in sys.path:
            sys.path.insert(0, REF)
        import flowpipe as fp

        model = fp.SeededMockModel(dim=dim, seed=0)
        emb = np.random.default_rng([seed, 2**32 - 1]).standard_normal(model.embed_dim)
        cond = fp.make_conditioning(embedding=emb)
        sched = fp.build_time_window_schedule(inference_steps=n)
        stamps = []
        t0 = time.perf_counter()
        res, _ = fp.run_stream(m, n, model, cond, seed, sched, dtype=dtype,
                               on_iteration=lambda st: stamps.append(time.perf_counter()))
        dt = time.perf_counter() - t0
        frames = len(res)
    else:  # oracle restatement (same algorithm, numpy)
        sys.path.insert(0, ROOT)
        from oracle import flowpipe_oracle as O

        sch = O.make_schedule(num_windows=4, steps=n)
        emb = np.random.default_rng([seed, 2**32 - 1]).standard_normal(8)
        stamps = []
        t0 = time.perf_counter()
        run = O.run_stream(m, n, lambda ids, ts, x: O.guided_mock_eps(0, ids, ts, emb, None, 1.0, dim), seed, sch, dim,
                           dtype=dtype)
        dt = time.perf_counter() - t0
        frames = len(run.order)
    # admission of generation g at iteration g, retirement at iteration g + n - 1
    lat = [1e3 * (stamps[g + n - 1] - (stamps[g - 1] if g > 0 else t0)) for g in range(m)] if stamps else []
    return dt, frames, lat


def time_reference_mock(m: int = 24, n: int = 4, dim: int = 16384, dtype: str = "f64", procs: int = 1,
                        seed: int = 1000) -> dict:
    """frames/s of `procs` independent streams (one per process) of m generations each."""
    use_ref = reference_available()
    jobs = [(m, n, dim, seed + p, dtype, use_ref) for p in range(procs)]
    t0 = time.perf_counter()
    if procs == 1:
        outs = [_one_stream(jobs[0])]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            outs = pool.map(_one_stream, jobs)
    wall = time.perf_counter() - t0
    frames = sum(o[1] for o in outs)
    lat = [x for o in outs for x in o[2]]
    return {"frames_per_s": frames / wall, "frames": frames, "wall_s": wall, "procs": procs,
            "p50_latency_ms": float(np.median(lat)) if lat else None,
            "kind": "reference" if use_ref else "port", "dtype": dtype,
            "sample": f"{procs} process(es) x 1 stream x {m} generations of n={n} at D={dim} ({dtype}), "
                      f"{'flowpipe.run_stream from baseline/_ref' if use_ref else 'oracle restatement'} + "
                      f"SeededMockModel"}
