"""CompiledEngine / adaptive_forward drop-in (reference engine.py), mirroring the
reference's tests/test_engine.py.  Dispatch logic and accounting are host-side
(CPU tests); the inner models compute on the GPU (gpu-marked tests)."""

import numpy as np
import pytest

import paper_2511_22009_b200 as sf

GRID = [0.0, 0.25, 0.5, 0.75]


def batch_at(ts, dim=4, rng=None):
    rng = rng or np.random.default_rng(0)
    ts = np.asarray(ts, dtype=np.float64)
    return sf.make_latent_batch(rng.standard_normal((len(ts), dim)), ts, np.arange(len(ts)))


def test_is_homogeneous():
    assert sf.is_homogeneous(np.array([0.5, 0.5]))
    assert sf.is_homogeneous(np.array([0.5, 0.5 + 1e-12]), eps=1e-6)
    assert not sf.is_homogeneous(np.array([0.5, 0.25]))
    assert sf.is_homogeneous(np.array([0.75]))
    with pytest.raises(sf.ParameterError):
        sf.is_homogeneous(np.array([]))


def test_engine_refuses_heterogeneous_directly():
    engine = sf.CompiledEngine(sf.SeededMockModel(dim=4))
    cond = sf.make_conditioning(np.zeros(8))
    with pytest.raises(sf.EngineRefusalError):
        engine.forward(batch_at([0.5, 0.25]), cond)
    assert engine.rejected == 1 and engine.invocations == 0


def test_engine_parameter_validation():
    model = sf.SeededMockModel(dim=4)
    with pytest.raises(sf.ParameterError):
        sf.CompiledEngine(model, per_call_overhead_us=-1.0)
    with pytest.raises(sf.ParameterError):
        sf.CompiledEngine(model, speed_factor=0.0)
    with pytest.raises(sf.ParameterError):
        sf.CompiledEngine(model, speed_factor=1.5)


@pytest.mark.gpu
def test_homogeneous_single_call_and_decomposition():
    model = sf.SeededMockModel(dim=4, seed=2)
    engine = sf.CompiledEngine(model)
    cond = sf.make_conditioning(np.zeros(8))
    sf.adaptive_forward(engine, batch_at([0.5, 0.5, 0.5]), cond)
    assert engine.invocations == 1 and engine.stats.calls_homogeneous == 1 and engine.stats.calls_decomposed == 0
    batch = batch_at([0.5, 0.25, 0.0])
    out = sf.adaptive_forward(engine, batch, cond)
    assert engine.invocations == 4 and engine.stats.calls_decomposed == 1
    assert np.array_equal(out.epsilon, model._compute(batch, cond).epsilon)


@pytest.mark.gpu
@pytest.mark.parametrize("make_model", [lambda: sf.AnalyticLinearModel(dim=6), lambda: sf.SeededMockModel(dim=6, seed=4)],
                         ids=["analytic", "mock"])
def test_dispatch_equivalence_random_batches(make_model):
    model = make_model()
    engine = sf.CompiledEngine(model)
    cond = sf.make_conditioning(np.zeros(8))
    rng = np.random.default_rng(41)
    for _ in range(30):
        b = int(rng.integers(1, 12))
        ts = np.full(b, rng.choice(GRID)) if rng.random() < 0.4 else rng.choice(GRID, size=b)
        batch = batch_at(ts, dim=6, rng=rng)
        before = engine.invocations
        out = sf.adaptive_forward(engine, batch, cond)
        assert np.array_equal(out.epsilon, model._compute(batch, cond).epsilon)
        assert engine.invocations - before == (1 if sf.is_homogeneous(ts, engine.eps) else b)


@pytest.mark.gpu
def test_aux_fieldwise_cost_accounting_and_order():
    model = sf.AnalyticLinearModel(dim=4, aux_scales=(0.5, 2.0))
    engine = sf.CompiledEngine(model)
    cond = sf.make_conditioning(np.zeros(8))
    batch = batch_at([0.75, 0.5, 0.0])
    out = sf.adaptive_forward(engine, batch, cond)
    for got, want in zip(out.aux, model._compute(batch, cond).aux):
        assert np.array_equal(got, want)
    mock = sf.SeededMockModel(dim=4, cost_us=100.0, seed=8)
    eng = sf.CompiledEngine(mock, per_call_overhead_us=7.0, speed_factor=0.3)
    sf.adaptive_forward(eng, batch_at([0.5, 0.25, 0.0, 0.75]), cond)
    per_call = 7.0 + 0.3 * 100.0
    assert eng.stats.total_simulated_time_us == pytest.approx(4 * per_call, rel=1e-12)
    ts = np.array([0.75, 0.0, 0.5, 0.25, 0.0])
    b2 = sf.make_latent_batch(np.zeros((5, 4)), ts, np.array([40, 30, 20, 10, 0]))
    assert np.array_equal(sf.adaptive_forward(eng, b2, cond).epsilon, mock._compute(b2, cond).epsilon)


@pytest.mark.gpu
def test_run_stream_through_compiled_engine_matches_plain_model():
    """pipeline.py:101-106: run_stream dispatches a CompiledEngine through adaptive_forward;
    the stream batch's mixed timesteps decompose, results are unchanged."""
    model = sf.SeededMockModel(dim=8, seed=2024)
    engine = sf.CompiledEngine(model)
    sched = sf.build_time_window_schedule(inference_steps=4)
    cond = sf.make_conditioning(np.zeros(8))
    er, es = sf.run_stream(6, 4, engine, cond, 77, sched)
    pr, ps = sf.run_stream(6, 4, model, cond, 77, sched)
    assert es.model_calls == ps.model_calls == 6 + 4 - 1
    for a, b in zip(er, pr):
        assert a.id == b.id and np.array_equal(a.latent, b.latent)
    assert engine.stats.calls_decomposed > 0 and engine.stats.calls_homogeneous > 0


@pytest.mark.gpu
def test_dit_engine_graph_replay_bit_exact():
    """The CUDA-graph engine over the DiT: homogeneous batches replay one graph per batch size,
    mixed batches replay the rows=1 graph per row; both bit-identical to inner._compute."""
    from paper_2511_22009_b200.dit import DIT_S2

    model = sf.DiTVelocityModel(DIT_S2, seed=12, max_rows=4, bias_std=0.02)
    engine = sf.CompiledEngine(model)
    rng = np.random.default_rng(5)
    cond = sf.make_conditioning(rng.standard_normal(8))
    for ts in ([0.5] * 4, [0.25, 0.75, 0.0], [0.5] * 6, [0.25] * 4, [0.0, 0.5]):
        x = rng.standard_normal((len(ts), model.dim)).astype(np.float32)
        batch = sf.make_latent_batch(x, np.asarray(ts), np.arange(len(ts)))
        out = sf.adaptive_forward(engine, batch, cond)
        assert np.array_equal(out.epsilon, model._compute(batch, cond).epsilon), ts
    gs = engine.graph_stats
    assert sorted(gs.sizes) == [1, 4, 6]  # one capture per batch size (6 rows = two launch sequences)
    assert gs.replays == engine.invocations == 1 + 3 + 1 + 1 + 2 and gs.eager_calls == 0
    assert engine.stats.calls_homogeneous == 3 and engine.stats.calls_decomposed == 2
