"""sf_numpy_normal (csrc/numpy_noise.cu) against numpy itself: the reference's
generation_noise (flowpipe src/pipeline.py:92-98) is
np.random.default_rng([seed, gen_id]).standard_normal(dim); the device rows must be
bit-identical in fp64 and equal to numpy's round-to-nearest fp32 cast."""

import numpy as np
import pytest
import torch

from paper_2511_22009_b200.errors import ParameterError
from paper_2511_22009_b200.pipeline import numpy_noise_device

pytestmark = pytest.mark.gpu


def _numpy(seeds, gen, dim):
    return np.stack([np.random.default_rng([int(s), gen]).standard_normal(dim) for s in seeds])


@pytest.mark.parametrize("gen", [0, 1, 977, 2**33 + 5])
def test_bit_identical_fp64(gen):
    seeds = list(range(64))  # 64 x 16384 draws: ~250 tail and ~7000 wedge resolutions
    got = numpy_noise_device(seeds, gen, 16384).cpu().numpy()
    want = _numpy(seeds, gen, 16384)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_large_seeds_and_fp32_cast():
    seeds = [0, 1, 2**31, 2**32 - 1, 2**32, 2**40 + 3, 2**62 + 11, 123456789012345]
    got = numpy_noise_device(seeds, 7, 4096, dtype=torch.float32).cpu().numpy()
    want = _numpy(seeds, 7, 4096).astype(np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("dim", [1, 7, 255, 256, 257, 1000])
def test_ragged_lengths(dim):
    seeds = [3, 4, 5]
    got = numpy_noise_device(seeds, 2, dim).cpu().numpy()
    assert np.array_equal(got.view(np.uint64), _numpy(seeds, 2, dim).view(np.uint64))


def test_prefix_property():
    """standard_normal(n) is a prefix of standard_normal(m > n) for the same generator."""
    a = numpy_noise_device([9], 4, 5000).cpu()
    b = numpy_noise_device([9], 4, 300).cpu()
    assert torch.equal(a[:, :300], b)


def test_errors():
    with pytest.raises(ValueError):
        numpy_noise_device([-1], 0, 16)
    with pytest.raises(ValueError):
        numpy_noise_device([1], -1, 16)
    with pytest.raises(ParameterError):
        numpy_noise_device([2**63], 0, 16)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_stream_batch_device_noise_equals_host_noise(dtype):
    """noise="numpy" (device generator) and noise="numpy_host" (numpy + upload) run the
    same multi-stream trajectories bit for bit."""
    import paper_2511_22009_b200 as sf

    sched = sf.build_time_window_schedule(inference_steps=4)
    model = sf.SeededMockModel(dim=4096, seed=3)
    cond = sf.make_conditioning(np.linspace(-1, 1, 8))
    outs = []
    for mode in ("numpy", "numpy_host"):
        sb = sf.StreamBatch(model, sched, 4, num_streams=3, cond=cond, seed=[11, 2**40, 0], m=5, dtype=dtype,
                            noise=mode)
        frames = []
        while not sb.done():
            frames += [(s, r.id, r.latent.copy()) for s, r in sb.step()]
        outs.append(frames)
    assert [(s, i) for s, i, _ in outs[0]] == [(s, i) for s, i, _ in outs[1]]
    for (_, _, a), (_, _, b) in zip(*outs):
        assert np.array_equal(a, b)


def test_c_abi_rejects_bad_arguments():
    from paper_2511_22009_b200 import _lib

    sd = torch.tensor([1], dtype=torch.int64, device="cuda")
    out = torch.empty(1, 8, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for args in ((sd.data_ptr(), 0, 1, 0, out.data_ptr(), _lib.SF_F64, st),    # D < 1
                 (sd.data_ptr(), -1, 1, 8, out.data_ptr(), _lib.SF_F64, st),   # gen < 0
                 (sd.data_ptr(), 0, 1, 8, out.data_ptr(), 7, st),              # dtype
                 (None, 0, 1, 8, out.data_ptr(), _lib.SF_F64, st)):            # null seeds
        with pytest.raises(ParameterError):
            _lib.call("sf_numpy_normal", *args)
