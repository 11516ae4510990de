"""AnalyticLinearModel (reference models.py:139-185) on the GPU (kernel K13).

eps_i = A x_i + t_i b in fp64, row by row.  The reference evaluates each row
with numpy's BLAS GEMV, whose summation order is not specified, so parity is
to round-off (rel 1e-12); row-decomposition invariance is bit-exact (the
property the reference's row-by-row loop exists for, models.py:142-146).
Pipeline equivalence mirrors the reference's acceptance criterion 2
(tests/test_acceptance.py:71-94, rel 1e-9) with the analytic model.
"""

import numpy as np
import pytest

from oracle import flowpipe_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sf():
    import paper_2511_22009_b200 as sf
    return sf


def _ref_eps(A, b, x, ts):
    return np.stack([A @ x[i].astype(np.float64) + ts[i] * b for i in range(len(ts))])


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_analytic_eps_matches_numpy(sf, dtype):
    rng = np.random.default_rng(3)
    D, B = 64, 5
    A = rng.standard_normal((D, D)) * 0.1
    b = rng.standard_normal(D)
    model = sf.AnalyticLinearModel(dim=D, a_matrix=A, b_vector=b)
    x = rng.standard_normal((B, D)).astype(dtype)
    ts = np.array([0.0, 0.25, 0.5, 0.75, 0.0])
    batch = sf.make_latent_batch(x, ts, np.arange(B))
    out = model.forward(batch, sf.make_conditioning(np.zeros(8))).epsilon
    np.testing.assert_allclose(out, _ref_eps(A, b, x, ts), rtol=1e-12, atol=1e-13)


def test_analytic_defaults_and_row_invariance(sf):
    D = 16
    model = sf.AnalyticLinearModel(dim=D)  # A = 0.1 I, b = 0.05 (models.py:162-165)
    rng = np.random.default_rng(4)
    x = rng.standard_normal((6, D))
    ts = np.linspace(0, 0.75, 6)
    cond = sf.make_conditioning(np.zeros(8))
    full = model.forward(sf.make_latent_batch(x, ts, np.arange(6)), cond).epsilon
    np.testing.assert_array_equal(full, 0.1 * x + ts[:, None] * 0.05)  # exact for the diagonal default
    for i in range(6):
        one = model.forward(sf.make_latent_batch(x[i:i + 1], ts[i:i + 1], np.arange(1)), cond).epsilon
        assert np.array_equal(one[0], full[i])


def test_analytic_shape_errors(sf):
    with pytest.raises(sf.ParameterError):
        sf.AnalyticLinearModel(dim=4, a_matrix=np.eye(3))
    with pytest.raises(sf.ParameterError):
        sf.AnalyticLinearModel(dim=4, b_vector=np.ones(3))


@pytest.mark.parametrize("m,n", [(1, 1), (4, 2), (9, 4), (5, 8)])
def test_stream_vs_vanilla_and_oracle_with_analytic(sf, m, n):
    rng = np.random.default_rng(m * 10 + n)
    D = 32
    A = rng.standard_normal((D, D)) * 0.05
    b = rng.standard_normal(D) * 0.1
    model = sf.AnalyticLinearModel(dim=D, a_matrix=A, b_vector=b)
    sched = sf.build_time_window_schedule(inference_steps=n)
    cond = sf.make_conditioning(np.zeros(8))
    sr, ss = sf.run_stream(m, n, model, cond, 77, sched)
    vr, vs = sf.run_vanilla(m, n, model, cond, 77, sched)
    assert ss.model_calls == m + n - 1 and vs.model_calls == m * n
    by_id = {r.id: r.latent for r in vr}
    osch = O.make_schedule(steps=n)
    run = O.run_stream(m, n, lambda ids, ts, x: _ref_eps(A, b, x, ts), 77, osch, D)
    for r in sr:
        scale = np.abs(by_id[r.id]).max()
        assert np.abs(r.latent - by_id[r.id]).max() <= 1e-9 * scale
        assert np.abs(r.latent - run.latents[r.id]).max() <= 1e-9 * scale


def test_reference_known_answers(sf):
    """Mirrors the reference's own tests/test_models.py:36-63 known answers."""
    cond = sf.make_conditioning(np.zeros(8))
    zero = sf.AnalyticLinearModel(dim=4, a_matrix=np.zeros((4, 4)), b_vector=np.zeros(4))
    out = zero.forward(sf.make_latent_batch(np.ones((3, 4)), [0.0, 0.25, 0.5], np.arange(3)), cond)
    assert np.all(out.epsilon == 0.0)
    m3 = sf.AnalyticLinearModel(dim=3)
    x = np.array([[1.0, -2.0, 4.0]])
    out = m3.forward(sf.make_latent_batch(x, [0.5], np.arange(1)), cond)
    np.testing.assert_allclose(out.epsilon, 0.1 * x + 0.5 * 0.05, rtol=1e-15)
    m2 = sf.AnalyticLinearModel(dim=2, a_matrix=np.array([[1.0, 2.0], [3.0, 4.0]]), b_vector=np.array([10.0, 20.0]))
    out2 = m2.forward(sf.make_latent_batch(np.array([[1.0, 1.0]]), [0.25], np.arange(1)), cond)
    assert out2.epsilon[0].tolist() == [1.0 + 2.0 + 2.5, 3.0 + 4.0 + 5.0]


def test_aux_outputs(sf):
    model = sf.AnalyticLinearModel(dim=6, aux_scales=(0.5, 2.0))
    cond = sf.make_conditioning(np.zeros(8))
    x = np.random.default_rng(0).standard_normal((2, 6))
    out = model.forward(sf.make_latent_batch(x, [0.0, 0.5], np.arange(2)), cond)
    assert len(out.aux) == 2
    np.testing.assert_array_equal(out.aux[0], 0.5 * out.epsilon)
    np.testing.assert_array_equal(out.aux[1], 2.0 * out.epsilon)
