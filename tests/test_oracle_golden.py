"""Pin the CPU oracle (oracle/flowpipe_oracle.py) before trusting it.

Two anchors, both from the reference:
1. the literal golden constants in the reference's own tests
   (pkg/tests/test_velocity.py:18-19, :101-108; test_schedule.py:20-21,
   :114-118; test_models.py:21-26; test_pipeline.py:18-22);
2. fixtures produced by importing the reference itself
   (tests/golden/make_golden.py -> flowpipe_golden.npz).
All comparisons are bit-exact (np.array_equal) unless the reference's own
test states a tolerance.
"""

import numpy as np
import pytest

from oracle import flowpipe_oracle as O

# reference literal goldens -------------------------------------------------
GOLDEN_T0 = 8.205887802938642  # test_velocity.py:18
ABAR_999 = 4.0358297653756754e-05  # test_schedule.py:21
ORACLE_T01 = (0.10975096295911049, 2.146611054504233, -1.2801861768771532)  # :114-118
MOCK_GOLDEN = [0.7420526547651705, -0.4957621902997431,
               -0.1268584068359535, 0.48547274159231946]  # test_models.py:21-26
VANILLA_GOLDENS = {  # test_pipeline.py:18-22
    0: [5.282935777121209, -23.854575690519436, 28.806230774069775, 24.918373768589632],
    1: [1.3742799518390016, 25.38791652452447, 17.457607583830363, 0.6042195561086086],
    2: [7.859996442343155, -17.485046967344623, 7.317959953020575, -12.8868935507846],
}
FROZEN_ROW0 = [17.2296240316625, 14.400724039047596, 14.181848017145596,
               -5.985559014737792, 7.335873677763303, -11.49212912159637]  # :101-108


def test_literal_goldens():
    s = O.make_schedule(steps=4)
    assert s.abar[0] == 0.9999
    assert s.abar[999] == pytest.approx(ABAR_999, rel=1e-12)
    x, tn = O.euler_step(np.full((1, 4), 0.1), np.full((1, 4), 1.0), [0.0], s)
    np.testing.assert_allclose(x[0], GOLDEN_T0, rtol=1e-12)
    assert tn[0] == 0.25
    x, tn = O.euler_step(np.full((1, 4), 0.1), np.full((1, 4), 1.0), [0.5], s)
    assert np.all(x == 1.0) and tn[0] == 0.75
    _, _, gamma, _, _, lam, eta = O.window_coeffs(0.1, s)
    assert gamma == pytest.approx(ORACLE_T01[0], rel=1e-12)
    assert lam == pytest.approx(ORACLE_T01[1], rel=1e-12)
    assert eta == pytest.approx(ORACLE_T01[2], rel=1e-12)
    eps = O.mock_eps(0, [0], [0.5], [np.zeros(8)], 4)
    assert eps[0].tolist() == MOCK_GOLDEN


def test_frozen_heterogeneous_row():
    s = O.make_schedule(steps=4)
    rng = np.random.default_rng(7)
    x = rng.standard_normal((3, 6))
    e = rng.standard_normal((3, 6))
    out, tn = O.euler_step(e, x, [0.0, 0.25, 0.5], s)
    np.testing.assert_allclose(out[0], FROZEN_ROW0, rtol=1e-12)
    assert np.array_equal(out[1], x[1]) and np.array_equal(out[2], x[2])
    assert tn.tolist() == [0.25, 0.5, 0.75]


def test_vanilla_goldens_through_oracle_stream():
    s = O.make_schedule(steps=2)
    emb = np.zeros(8)
    fn = lambda ids, ts, x: O.guided_mock_eps(5, ids, ts, emb, None, 1.0, 4)  # noqa: E731
    run = O.run_stream(3, 2, fn, 42, s, 4)
    assert run.order == [0, 1, 2]
    for g, want in VANILLA_GOLDENS.items():
        np.testing.assert_allclose(run.latents[g], want, rtol=1e-12)


@pytest.mark.parametrize("k", [1, 3, 4, 5])
def test_window_params_match_reference(golden, k):
    s = O.make_schedule(num_windows=k, steps=4)
    ts = golden[f"wp_K{k}_t"]
    names = ("t_s", "t_e", "gamma", "lambda_s", "eta_s", "lambda_t", "eta_t")
    for i, t in enumerate(ts):
        got = O.window_coeffs(float(t), s)
        for name, v in zip(names, got):
            assert v == golden[f"wp_K{k}_{name}"][i], (name, t)


def test_abar_and_successor(golden):
    assert np.array_equal(O.noise_table(), golden["abar_default"])
    for n in (1, 2, 3, 4, 8):
        s = O.make_schedule(steps=n)
        got = [O.grid_successor(float(t), s) for t in s.grid]
        assert got == golden[f"next_n{n}"].tolist()


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("n", [4, 8])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_batched_step_bit_exact(golden, k, n, dt):
    key = f"step_K{k}_n{n}_{dt}"
    s = O.make_schedule(num_windows=k, steps=n)
    out, tn = O.euler_step(golden[key + "_eps"], golden[key + "_x"], golden[key + "_t"], s)
    assert out.dtype == golden[key + "_out"].dtype
    assert np.array_equal(out, golden[key + "_out"])
    assert np.array_equal(tn, golden[key + "_tnext"])


def test_mock_rows_bit_exact(golden):
    ids, ts = golden["mock_ids"], golden["mock_ts"]
    emb, neg = golden["mock_emb"], golden["mock_neg"]
    keys = [O.mock_row_key(42, int(i), float(t), emb) for i, t in zip(ids, ts)]
    assert np.array_equal(np.array(keys, np.uint64), golden["mock_keys"])
    assert np.array_equal(O.guided_mock_eps(42, ids, ts, emb, None, 1.0, 64),
                          golden["mock_eps_plain"])
    assert np.array_equal(O.guided_mock_eps(42, ids, ts, emb, neg, 7.5, 64),
                          golden["mock_eps_cfg"])
    assert np.array_equal(O.guided_mock_eps(42, ids, ts, emb, None, 3.0, 64),
                          golden["mock_eps_cfg_zero_neg"])


def test_run_stream_bit_exact(golden):
    for name in golden["run_cases"]:
        m, n, k, d, seed, mseed, f32 = golden[name + "_meta"].tolist()
        w = float(golden[name + "_w"][0])
        emb = golden[name + "_emb"]
        s = O.make_schedule(num_windows=k, steps=n)
        fn = lambda ids, ts, x: O.guided_mock_eps(mseed, ids, ts, emb, None, w, d)  # noqa
        run = O.run_stream(m, n, fn, seed, s, d, dtype=np.float32 if f32 else np.float64)
        assert run.order == golden[name + "_order"].tolist()
        assert [run.spans[g] for g in run.order] == golden[name + "_spans"].tolist()
        got = np.stack([run.latents[g] for g in run.order])
        assert np.array_equal(got, golden[name + "_latents"]), name
        counts = [run.model_calls, run.scheduler_calls, run.param_evals, run.decodes]
        assert counts == golden[name + "_counts"].tolist()
        assert sum(run.batch_ids, []) == golden[name + "_q_ids"].tolist()
        assert sum(run.batch_ts, []) == golden[name + "_q_ts"].tolist()
