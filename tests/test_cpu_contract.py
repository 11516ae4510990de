"""CPU-side contract tests (no GPU needed).

* libstreamflow.so loads and exports every symbol include/streamflow.h declares;
* host-side argument validation mirrors the reference (schedule.py:47-173,
  velocity.py:47-69, models.py:58-73, pipeline.py:128-136), raising the same
  exception classes;
* with no CUDA device every compute entry point raises (no CPU fallback).
"""

import ctypes
import os
import subprocess

import numpy as np
import pytest
import torch

import paper_2511_22009_b200 as sf
from paper_2511_22009_b200 import _lib


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert b"sm_100a" in _lib.fn("sf_version")()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_library_contains_tcgen05_and_tma():
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA loads
    assert "LDTM" in sass     # tcgen05.ld (TMEM -> registers)
    # The network's GEMMs and attention are tcgen05; the legacy mma.sync path appears only in the
    # two thin 16-wide projections (patch embed K=16, final layer N=16), where it is HBM-bound.
    hmma_funcs = set()
    func = None
    for line in sass.splitlines():
        if "Function :" in line:
            func = line.split("Function :")[1].strip()
        elif "HMMA" in line.replace("UTCHMMA", "") and func:
            hmma_funcs.add(func)
    assert hmma_funcs, "expected the mma.sync patch-embed / final-layer kernels"
    assert all("patch_embed_ln_mma_kernel" in f or "final_layer_mma_kernel" in f for f in hmma_funcs), hmma_funcs


@pytest.mark.parametrize("kwargs", [dict(beta_start=0.0), dict(beta_start=0.3, beta_end=0.2),
                                    dict(beta_end=1.0), dict(t_max=1)])
def test_noise_schedule_validation(kwargs):
    with pytest.raises(sf.ParameterError):
        sf.build_noise_schedule(**{"t_max": 10, "beta_start": 1e-4, "beta_end": 0.02, **kwargs})


@pytest.mark.parametrize("bad", [dict(boundaries=[0.1, 0.5, 1.0]), dict(boundaries=[0.0, 0.5, 0.4, 1.0]),
                                 dict(eps=-1e-6), dict(eps=0.2), dict(inference_grid=[0.0, 0.5, 0.5]),
                                 dict(inference_grid=[0.0, 1.5]), dict(num_windows=0)])
def test_window_schedule_validation(bad):
    with pytest.raises(sf.ParameterError):
        sf.build_time_window_schedule(**bad)


def test_schedule_tables_match_reference_goldens(golden):
    s = sf.build_time_window_schedule(inference_steps=4)
    assert np.array_equal(s.noise_schedule.alphas_cumprod, golden["abar_default"])
    assert sf.uniform_inference_grid(4).tolist() == [0.0, 0.25, 0.5, 0.75]
    assert sf.build_noise_schedule(t_max=2, beta_start=0.5, beta_end=0.5).alphas_cumprod.tolist() == [0.5, 0.25]


def test_latent_batch_and_conditioning_validation():
    with pytest.raises(sf.ParameterError):
        sf.make_latent_batch(np.zeros((2, 4)), [0.0], [0, 1])
    with pytest.raises(sf.ParameterError):
        sf.make_latent_batch(np.zeros((2, 4)), [0.0, 1.5], [0, 1])
    with pytest.raises(sf.ParameterError):
        sf.make_latent_batch(np.zeros(4), [0.0], [0])
    with pytest.raises(sf.ParameterError):
        sf.make_conditioning(np.zeros(8), guidance_scale=-0.5)
    with pytest.raises(sf.ParameterError):
        sf.make_conditioning(np.zeros(8), negative_embedding=np.zeros(5))
    b = sf.make_latent_batch(np.zeros((2, 4)), [0.0, 0.25], [7, 9])
    c = sf.make_conditioning(np.ones(8), guidance_scale=7.5, negative_embedding=np.full(8, -1.0))
    d2, c2 = sf.apply_cfg(b, c)  # host-side doubling (models.py:244-275)
    assert d2.batch_size == 4 and d2.ids.tolist() == [7, 9, 7, 9]
    assert np.all(c2.row_embeddings[:2] == -1.0) and np.all(c2.row_embeddings[2:] == 1.0)
    assert sf.apply_cfg(b, sf.make_conditioning(np.ones(8)))[0] is b


def test_exception_hierarchy_matches_reference():
    assert issubclass(sf.ParameterError, ValueError) and issubclass(sf.TimeDomainError, ValueError)
    assert issubclass(sf.StateError, RuntimeError) and issubclass(sf.InvariantError, RuntimeError)
    assert issubclass(sf.EngineRefusalError, sf.StateError)
    for e in (sf.ParameterError, sf.TimeDomainError, sf.StateError, sf.InvariantError, sf.ConfigError):
        assert issubclass(e, sf.FlowPipeError)


def test_c_abi_rejects_bad_arguments_without_touching_the_device():
    # argument validation happens before any launch
    assert _lib.fn("sf_velocity_step")(None, 7, None, None, 7, None, 1, 1, None) == _lib.SF_ERR_PARAMETER
    assert _lib.fn("sf_gemm_bf16")(None, None, None, None, 128, 100, 64, 0, None) == _lib.SF_ERR_PARAMETER
    assert _lib.fn("sf_attention")(None, None, None, None, 1, 6, 1000, None) == _lib.SF_ERR_PARAMETER
    assert _lib.fn("sf_mock_keys")(0, None, None, None, 1, 0, None, None) == _lib.SF_ERR_PARAMETER


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    sched = sf.build_time_window_schedule(inference_steps=2)
    model = sf.SeededMockModel(dim=4, seed=5)
    with pytest.raises(Exception):
        sf.run_stream(3, 2, model, sf.make_conditioning(np.zeros(8)), 42, sched)
    with pytest.raises(Exception):
        sf.batched_velocity_step(np.zeros((1, 4)), sf.make_latent_batch(np.zeros((1, 4)), [0.0], [0]), sched)
    with pytest.raises(RuntimeError):
        sf.DiTVelocityModel(max_rows=1)
    with pytest.raises(RuntimeError):
        sf.StreamBatch(model, sched, 2, cond=sf.make_conditioning(np.zeros(8)))
