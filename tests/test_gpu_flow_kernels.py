"""K1 / K10-lite / K12 kernels through the C ABI, bit-exact against the
reference fixtures (tests/golden/flowpipe_golden.npz) and the oracle."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import flowpipe_oracle as O

pytestmark = pytest.mark.gpu


def L():
    from paper_2511_22009_b200 import _lib
    return _lib


def stream():
    return torch.cuda.current_stream().cuda_stream


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def sched_struct(k, n, keep):
    s = O.make_schedule(num_windows=k, steps=n)
    b, a, g = dev(s.boundaries), dev(s.abar), dev(s.grid)
    keep += [b, a, g]
    return L().SfSchedule(b.data_ptr(), a.data_ptr(), g.data_ptr(), k, len(s.abar), n, 0, s.eps), s


@pytest.mark.parametrize("k", [1, 3, 4, 5])
def test_window_params_bit_exact(golden, k):
    keep = []
    st, s = sched_struct(k, 4, keep)
    ts = golden[f"wp_K{k}_t"]
    out = torch.empty(len(ts), 12, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    tsd = dev(ts)
    L().call("sf_window_params", C.byref(st), tsd.data_ptr(), len(ts), out.data_ptr(),
             status.data_ptr(), stream())
    o = out.cpu().numpy()
    names = {"t_s": 2, "t_e": 3, "gamma": 4, "lambda_s": 5, "eta_s": 6, "lambda_t": 7, "eta_t": 8}
    for name, col in names.items():
        assert np.array_equal(o[:, col], golden[f"wp_K{k}_{name}"]), name
    # random t are off-grid -> status flag set
    assert status.item() & 2


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("n", [4, 8])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_velocity_step_bit_exact(golden, k, n, dt):
    keep = []
    st, s = sched_struct(k, n, keep)
    key = f"step_K{k}_n{n}_{dt}"
    x, e, ts = golden[key + "_x"], golden[key + "_eps"], golden[key + "_t"]
    B, D = x.shape
    params = torch.empty(B, 12, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    tsd = dev(ts)
    L().call("sf_window_params", C.byref(st), tsd.data_ptr(), B, params.data_ptr(),
             status.data_ptr(), stream())
    xd, ed = dev(x), dev(e)
    out = torch.empty_like(xd)
    code = 1 if dt == "f64" else 0
    L().call("sf_velocity_step", ed.data_ptr(), code, xd.data_ptr(), out.data_ptr(), code,
             params.data_ptr(), B, D, stream())
    assert status.item() == 0
    assert np.array_equal(out.cpu().numpy(), golden[key + "_out"])
    assert np.array_equal(params[:, 1].cpu().numpy(), golden[key + "_tnext"])


def test_mock_keys_and_eps_bit_exact(golden):
    ids, ts, emb = golden["mock_ids"], golden["mock_ts"], golden["mock_emb"]
    B = len(ids)
    embs = dev(np.tile(emb, (B, 1)))
    keys = torch.empty(B, dtype=torch.int64, device="cuda")
    idd, tsd = dev(ids), dev(ts)
    L().call("sf_mock_keys", 42, idd.data_ptr(), tsd.data_ptr(), embs.data_ptr(), B, 8,
             keys.data_ptr(), stream())
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), golden["mock_keys"])
    out = torch.empty(B, 64, dtype=torch.float64, device="cuda")
    L().call("sf_mock_eps", keys.data_ptr(), B, 64, out.data_ptr(), stream())
    assert np.array_equal(out.cpu().numpy(), golden["mock_eps_plain"])
