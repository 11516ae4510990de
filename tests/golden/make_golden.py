"""Generate golden fixtures by importing the UNMODIFIED reference ``flowpipe``.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py

It writes ``tests/golden/flowpipe_golden.npz``.  The GPU box never reads
``/root/reference``; tests there use only the committed ``.npz``.

Cases:
* window coefficients / successor at dense t for K in {1, 3, 4, 5} and the
  flat alpha-bar table  (schedule.py:224-295)
* batched_velocity_step on random heterogeneous batches, fp64 + fp32,
  K in {3, 4}  (velocity.py:93-135)
* SeededMockModel rows incl. CFG doubling  (models.py:188-296)
* run_stream end to end: final latents, completion order, per-iteration
  batch ids/timesteps, counters; small D for many (m, n, K, w, dtype)
  combos and D = 16384 (64x64x4 latent) for the headline shape
  (pipeline.py:139-220)
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import flowpipe as fp  # noqa: E402
from flowpipe.models import SeededMockModel  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "flowpipe_golden.npz")


class RecordingMock(SeededMockModel):
    """Records (ids, timesteps) of every forward: the queue-order witness."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.calls = []

    def _compute(self, batch, cond):
        self.calls.append((batch.ids.copy(), batch.timesteps.copy()))
        return super()._compute(batch, cond)


def sched_for(k, n):
    return fp.build_time_window_schedule(num_windows=k, inference_steps=n)


def main():
    g = {}
    # --- window coefficients ------------------------------------------------
    rng = np.random.default_rng(2511)
    ts_dense = np.concatenate([rng.uniform(0, 1, 200), np.linspace(0, 1, 41)])
    for k in (1, 3, 4, 5):
        s = sched_for(k, 4)
        wp = fp.window_params(ts_dense, s)
        g[f"wp_K{k}_t"] = ts_dense
        for name in ("t_s", "t_e", "gamma", "lambda_s", "eta_s", "lambda_t", "eta_t"):
            g[f"wp_K{k}_{name}"] = getattr(wp, name)
    for n in (1, 2, 3, 4, 8):
        s = sched_for(4, n)
        g[f"next_n{n}"] = fp.next_timestep(s.inference_grid, s)
    g["abar_default"] = fp.build_noise_schedule().alphas_cumprod

    # --- batched velocity step -----------------------------------------------
    for k in (3, 4):
        for n in (4, 8):
            s = sched_for(k, n)
            for dt in ("f64", "f32"):
                r = np.random.default_rng(100 * k + n + (dt == "f32"))
                b, d = 37, 24
                ts = r.choice(s.inference_grid, size=b)
                x = r.standard_normal((b, d))
                e = r.standard_normal((b, d))
                if dt == "f32":
                    x = x.astype(np.float32)
                    e = e.astype(np.float32)
                out = fp.batched_velocity_step(
                    e, fp.LatentBatch(data=x, timesteps=ts, ids=np.arange(b)), s)
                key = f"step_K{k}_n{n}_{dt}"
                g[key + "_x"] = x
                g[key + "_eps"] = e
                g[key + "_t"] = ts
                g[key + "_out"] = out.data
                g[key + "_tnext"] = out.timesteps

    # --- mock model rows ------------------------------------------------------
    r = np.random.default_rng(77)
    emb = r.standard_normal(8)
    neg = r.standard_normal(8)
    ids = np.array([0, 1, 5, 12345, 7, 3], dtype=np.int64)
    ts = np.array([0.0, 0.25, 0.5, 0.75, 0.3333333333333333, 1.0])
    model = SeededMockModel(dim=64, seed=42)
    batch = fp.make_latent_batch(np.zeros((6, 64)), ts, ids)
    g["mock_ids"], g["mock_ts"], g["mock_emb"], g["mock_neg"] = ids, ts, emb, neg
    g["mock_eps_plain"] = model.forward(batch, fp.make_conditioning(emb)).epsilon
    cond = fp.make_conditioning(emb, guidance_scale=7.5, negative_embedding=neg)
    d2, c2 = fp.apply_cfg(batch, cond)
    g["mock_eps_cfg"] = fp.handle_cfg(model.forward(d2, c2), 7.5).epsilon
    cond0 = fp.make_conditioning(emb, guidance_scale=3.0)
    d2, c2 = fp.apply_cfg(batch, cond0)
    g["mock_eps_cfg_zero_neg"] = fp.handle_cfg(model.forward(d2, c2), 3.0).epsilon
    keys = np.array([model._row_key(int(i), float(t), emb) for i, t in zip(ids, ts)],
                    dtype=np.uint64)
    g["mock_keys"] = keys

    # --- run_stream end to end -------------------------------------------------
    cases = []
    for (m, n, k, w, dt, d) in [
        (3, 2, 4, 1.0, "f64", 4), (7, 4, 4, 1.0, "f64", 16), (7, 4, 3, 1.0, "f64", 16),
        (5, 4, 3, 7.5, "f64", 16), (9, 8, 3, 7.5, "f64", 8), (6, 1, 3, 2.0, "f64", 8),
        (4, 3, 5, 1.0, "f32", 16), (5, 4, 3, 7.5, "f32", 16), (2, 4, 3, 1.0, "f64", 16),
        (6, 4, 3, 7.5, "f64", 16384), (6, 4, 4, 1.0, "f32", 16384), (5, 2, 1, 7.5, "f64", 32),
    ]:
        name = f"run_m{m}_n{n}_K{k}_w{w}_{dt}_D{d}"
        s = sched_for(k, n)
        seed = 1000 + m * 10 + n
        model = RecordingMock(dim=d, seed=seed % 97)
        emb = np.random.default_rng([seed, 2**32 - 1]).standard_normal(8)
        cond = fp.make_conditioning(emb, guidance_scale=w)
        res, st = fp.run_stream(m, n, model, cond, seed, s,
                                dtype=np.float32 if dt == "f32" else np.float64)
        cases.append(name)
        g[name + "_meta"] = np.array([m, n, k, d, seed, seed % 97, dt == "f32"], np.int64)
        g[name + "_w"] = np.array([w])
        g[name + "_emb"] = emb
        g[name + "_order"] = np.array([x.id for x in res], np.int64)
        g[name + "_spans"] = np.array([x.iterations_spanned for x in res], np.int64)
        g[name + "_latents"] = np.stack([x.latent for x in res])
        g[name + "_counts"] = np.array([st.model_calls, st.scheduler_calls,
                                        st.step_stats.param_evals, st.decodes], np.int64)
        # queue witness: only the first half of CFG-doubled calls (ids repeat)
        ids_flat, ts_flat, lens = [], [], []
        for ids_c, ts_c in model.calls:
            h = len(ids_c) // 2 if w != 1.0 else len(ids_c)
            ids_flat += ids_c[:h].tolist()
            ts_flat += ts_c[:h].tolist()
            lens.append(h)
        g[name + "_q_ids"] = np.array(ids_flat, np.int64)
        g[name + "_q_ts"] = np.array(ts_flat)
        g[name + "_q_lens"] = np.array(lens, np.int64)
    g["run_cases"] = np.array(cases)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
