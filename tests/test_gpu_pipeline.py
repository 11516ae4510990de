"""Drop-in pipeline API on the GPU vs the reference (bit-exact).

Fixtures come from the reference itself (tests/golden/make_golden.py); the
oracle (oracle/flowpipe_oracle.py) covers multi-stream cases.  Mirrors the
reference's own tests: pkg/tests/test_pipeline.py (goldens :18-22, call
counts :43-59, equivalence :98-110, queue invariants :119-151, fp32
:195-202), test_velocity.py and test_models.py.
"""

import numpy as np
import pytest

from oracle import flowpipe_oracle as O

pytestmark = pytest.mark.gpu

VANILLA_GOLDENS = {  # reference pkg/tests/test_pipeline.py:18-22
    0: [5.282935777121209, -23.854575690519436, 28.806230774069775, 24.918373768589632],
    1: [1.3742799518390016, 25.38791652452447, 17.457607583830363, 0.6042195561086086],
    2: [7.859996442343155, -17.485046967344623, 7.317959953020575, -12.8868935507846],
}


@pytest.fixture(scope="module")
def sf():
    import paper_2511_22009_b200 as sf
    return sf


def test_vanilla_goldens_through_stream(sf):
    sched = sf.build_time_window_schedule(inference_steps=2)
    model = sf.SeededMockModel(dim=4, seed=5)
    cond = sf.make_conditioning(np.zeros(8))
    res, stats = sf.run_stream(3, 2, model, cond, 42, sched)
    assert [r.id for r in res] == [0, 1, 2]
    for r in res:
        np.testing.assert_allclose(r.latent, VANILLA_GOLDENS[r.id], rtol=1e-12)
    vres, vstats = sf.run_vanilla(3, 2, model, cond, 42, sched)
    for r in vres:
        np.testing.assert_allclose(r.latent, VANILLA_GOLDENS[r.id], rtol=1e-12)
    assert stats.model_calls == 4 and vstats.model_calls == 6


def test_run_stream_bit_exact_vs_reference_fixtures(sf, golden):
    for name in golden["run_cases"]:
        m, n, k, d, seed, mseed, f32 = golden[name + "_meta"].tolist()
        w = float(golden[name + "_w"][0])
        sched = sf.build_time_window_schedule(num_windows=k, inference_steps=n)
        model = sf.SeededMockModel(dim=d, seed=mseed)
        cond = sf.make_conditioning(golden[name + "_emb"], guidance_scale=w)
        res, st = sf.run_stream(m, n, model, cond, seed, sched, dtype=np.float32 if f32 else np.float64)
        assert [r.id for r in res] == golden[name + "_order"].tolist(), name
        assert [r.iterations_spanned for r in res] == golden[name + "_spans"].tolist()
        got = np.stack([r.latent for r in res])
        want = golden[name + "_latents"]
        assert got.dtype == want.dtype
        assert np.array_equal(got, want), (name, np.abs(got - want).max())
        counts = [st.model_calls, st.scheduler_calls, st.step_stats.param_evals, st.decodes]
        assert counts == golden[name + "_counts"].tolist(), name


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("w", [1.0, 7.5])
def test_multi_stream_batch_matches_independent_runs(sf, dtype, w):
    """S streams in one device batch == S independent reference runs."""
    S, m, n, k, D = 5, 6, 4, 3, 256
    sched = sf.build_time_window_schedule(num_windows=k, inference_steps=n)
    model = sf.SeededMockModel(dim=D, seed=9)
    rng = np.random.default_rng(0)
    embs = [rng.standard_normal(8) for _ in range(S)]
    negs = [rng.standard_normal(8) for _ in range(S)]
    conds = [sf.make_conditioning(embs[s], guidance_scale=w, negative_embedding=negs[s]) for s in range(S)]
    sb = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=100, m=m, dtype=dtype)
    out = sb()
    osch = O.make_schedule(num_windows=k, steps=n)
    for s in range(S):
        fn = lambda ids, ts, x, s=s: O.guided_mock_eps(9, ids, ts, embs[s], negs[s], w, D)  # noqa: E731
        run = O.run_stream(m, n, fn, 100 + s, osch, D, dtype=dtype)
        assert [r.id for r in out[s]] == run.order
        for r in out[s]:
            assert np.array_equal(r.latent, run.latents[r.id])
        assert sb.stats[s].step_stats.param_evals == m * n


def test_queue_invariants(sf):
    """pkg/tests/test_pipeline.py:119-151."""
    m, n = 7, 4
    sched = sf.build_time_window_schedule(inference_steps=n)
    model = sf.SeededMockModel(dim=16, seed=1)
    seen = []
    sf.run_stream(m, n, model, sf.make_conditioning(np.zeros(8)), 1, sched, on_iteration=seen.append)
    assert len(seen) == m + n - 1
    for state in seen:
        j = state.iteration
        assert state.emitted == max(0, j - n + 2)
        offset = max(0, j - m + 1)
        for p, entry in enumerate(state.buffer):
            assert entry.stage == p + 1 + offset
        if n - 2 <= j < m:
            assert len(state.buffer) == n - 1


def test_batched_velocity_step_dropin(sf, golden):
    for k in (3, 4):
        for n in (4, 8):
            for dt in ("f64", "f32"):
                key = f"step_K{k}_n{n}_{dt}"
                s = sf.build_time_window_schedule(num_windows=k, inference_steps=n)
                b = sf.LatentBatch(data=golden[key + "_x"], timesteps=golden[key + "_t"],
                                   ids=np.arange(len(golden[key + "_t"])))
                stats = sf.StepStats()
                out = sf.batched_velocity_step(golden[key + "_eps"], b, s, stats)
                assert np.array_equal(out.data, golden[key + "_out"])
                assert np.array_equal(out.timesteps, golden[key + "_tnext"])
                assert stats.param_evals == b.batch_size and stats.elementwise_ops == 3


def test_errors_match_reference(sf):
    s = sf.build_time_window_schedule(inference_steps=4)
    b = sf.make_latent_batch(np.zeros((1, 4)), [0.4], [0])
    with pytest.raises(sf.TimeDomainError):
        sf.batched_velocity_step(np.zeros((1, 4)), b, s)
    with pytest.raises(sf.ParameterError):
        sf.batched_velocity_step(np.zeros((1, 5)), b, s)
    with pytest.raises(sf.TimeDomainError):
        sf.next_timestep([0.3], s)
    with pytest.raises(sf.StateError):
        sf.handle_cfg(sf.ModelOutput(epsilon=np.zeros((3, 2))), 2.0)
    model = sf.SeededMockModel(dim=4)
    with pytest.raises(sf.ParameterError):
        sf.run_stream(0, 2, model, sf.make_conditioning(np.zeros(8)), 0, s)
    with pytest.raises(sf.ParameterError):
        sf.run_stream(2, 8, model, sf.make_conditioning(np.zeros(8)), 0, s)


def test_window_params_and_mock_model_dropin(sf, golden):
    s = sf.build_time_window_schedule(num_windows=3, inference_steps=4)
    wp = sf.window_params(golden["wp_K3_t"], s)
    assert np.array_equal(wp.lambda_t, golden["wp_K3_lambda_t"])
    assert np.array_equal(wp.eta_t, golden["wp_K3_eta_t"])
    model = sf.SeededMockModel(dim=64, seed=42)
    batch = sf.make_latent_batch(np.zeros((6, 64)), golden["mock_ts"], golden["mock_ids"])
    cond = sf.make_conditioning(golden["mock_emb"], guidance_scale=7.5, negative_embedding=golden["mock_neg"])
    d2, c2 = sf.apply_cfg(batch, cond)
    out = sf.handle_cfg(model.forward(d2, c2), 7.5)
    assert np.array_equal(out.epsilon, golden["mock_eps_cfg"])


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_mixed_guidance_scales_match_independent_runs(sf, dtype):
    """Streams with different guidance scales (1.0 = unguided, as independent run_stream calls may
    have) in ONE device batch == independent reference runs, bit for bit (per-stream w in the
    fused step; a w == 1 stream takes its conditional eps unchanged)."""
    S, m, n, k, D = 4, 5, 3, 4, 128
    ws = [1.0, 7.5, 2.0, 1.0]
    sched = sf.build_time_window_schedule(num_windows=k, inference_steps=n)
    model = sf.SeededMockModel(dim=D, seed=4)
    rng = np.random.default_rng(9)
    embs = [rng.standard_normal(8) for _ in range(S)]
    conds = [sf.make_conditioning(embs[s], guidance_scale=ws[s]) for s in range(S)]
    sb = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=300, m=m, dtype=dtype)
    out = sb()
    osch = O.make_schedule(num_windows=k, steps=n)
    for s in range(S):
        fn = lambda ids, ts, x, s=s: O.guided_mock_eps(4, ids, ts, embs[s], None, ws[s], D)  # noqa: E731
        run = O.run_stream(m, n, fn, 300 + s, osch, D, dtype=dtype)
        for r in out[s]:
            assert np.array_equal(r.latent, run.latents[r.id]), (s, r.id)


def _random_cases(count=40, seed=2026):
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(count):
        S = int(rng.integers(1, 8))
        n = int(rng.integers(1, 6))
        k = int(rng.integers(1, 6))
        m = int(rng.integers(1, 10))
        D = int(rng.choice([8, 100, 256, 1000, 4096]))
        dtype = np.float64 if rng.random() < 0.5 else np.float32
        ws = [1.0 if rng.random() < 0.4 else float(np.round(rng.uniform(0.0, 9.0), 3)) for _ in range(S)]
        has_neg = [bool(rng.random() < 0.5) for _ in range(S)]
        seeds = [int(v) for v in rng.integers(0, 2**31, size=S)]  # arbitrary, non-consecutive
        cases.append((i, S, n, k, m, D, dtype, ws, has_neg, seeds))
    return cases


@pytest.mark.parametrize("case", _random_cases(), ids=lambda c: f"case{c[0]}")
def test_random_stream_batches_match_oracle(sf, case):
    """Seeded random configurations (streams, steps per generation, windows, generations, latent
    size, dtype, per-stream guidance with and without negative embeddings, arbitrary per-stream
    seeds): one device batch == independent oracle runs, bit for bit, with the reference's
    call counts."""
    _, S, n, k, m, D, dtype, ws, has_neg, seeds = case
    sched = sf.build_time_window_schedule(num_windows=k, inference_steps=n)
    model = sf.SeededMockModel(dim=D, seed=17)
    rng = np.random.default_rng(seeds[0] % 1000)
    embs = [rng.standard_normal(8) for _ in range(S)]
    negs = [rng.standard_normal(8) if has_neg[s] else None for s in range(S)]
    conds = [sf.make_conditioning(embs[s], guidance_scale=ws[s], negative_embedding=negs[s]) for s in range(S)]
    sb = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=seeds, m=m, dtype=dtype)
    out = sb()
    osch = O.make_schedule(num_windows=k, steps=n)
    for s in range(S):
        fn = lambda ids, ts, x, s=s: O.guided_mock_eps(17, ids, ts, embs[s], negs[s], ws[s], D)  # noqa: E731
        run = O.run_stream(m, n, fn, seeds[s], osch, D, dtype=dtype)
        assert [r.id for r in out[s]] == run.order, s
        for r in out[s]:
            assert r.latent.dtype == dtype
            assert np.array_equal(r.latent, run.latents[r.id]), (s, r.id)
        st = sb.stats[s]
        assert st.step_stats.param_evals == m * n
        assert st.model_calls == m + n - 1 and st.decodes == m
