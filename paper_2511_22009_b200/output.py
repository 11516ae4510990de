"""Result output in the reference's on-disk format (flowpipe cli.py:60-95).

``generate`` is the reference's ``flowpipe generate`` path (cli.py:60-95,
config.py:255-289: mock or analytic model, seed-derived conditioning
embedding, default schedule, one ``run_stream``) on the device pipeline;
``results_csv`` renders results exactly like the reference (``id,dim,values...``
header, ``repr`` floats), so the bytes match the reference's for the same
arguments (acceptance C8, tests/test_acceptance.py:224-231).
"""

from __future__ import annotations

import numpy as np

from .engine import CompiledEngine
from .models import AnalyticLinearModel, SeededMockModel, make_conditioning
from .pipeline import run_stream
from .schedule import build_time_window_schedule

_CONDITIONING_STREAM = 2**32 - 1  # config.py:50-51 sub-seed of the conditioning embedding


def results_csv(results) -> str:
    """cli.py:83-88: one line per generation, ``id,dim,v0,v1,...`` with repr floats."""
    lines = ["id,dim,values..."]
    for r in results:
        lat = np.asarray(r.latent)
        lines.append(f"{r.id},{len(lat)}," + ",".join(repr(float(v)) for v in lat))
    return "\n".join(lines) + "\n"


def write_results_csv(results, path: str) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(results_csv(results))


def generate(num_images: int = 4, steps: int = 4, seed: int = 0, guidance: float = 1.0, dtype: str = "float64",
             model: str = "mock", dim: int = 16, cost_us_per_call: float = 0.0, engine: str = "none",
             num_windows: int = 4, out: str | None = None) -> str:
    """The reference's ``generate`` command (defaults = its config defaults) -> CSV text."""
    inner = (AnalyticLinearModel(dim=dim, cost_us=cost_us_per_call) if model == "analytic"
             else SeededMockModel(dim=dim, cost_us=cost_us_per_call, seed=seed))
    runner = CompiledEngine(inner) if engine == "compiled" else inner
    emb = np.random.default_rng([seed, _CONDITIONING_STREAM]).standard_normal(inner.embed_dim)
    cond = make_conditioning(emb, guidance_scale=guidance)
    sched = build_time_window_schedule(num_windows=num_windows, inference_steps=steps)
    results, _ = run_stream(num_images, steps, runner, cond, seed, sched,
                            dtype=np.float32 if dtype == "float32" else np.float64)
    text = results_csv(results)
    if out is not None:
        with open(out, "w", encoding="utf-8") as fh:
            fh.write(text)
    return text
