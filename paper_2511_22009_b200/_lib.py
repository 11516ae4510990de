"""ctypes binding of ``libstreamflow.so`` (the C ABI in ``include/streamflow.h``).

There is no fallback: if the library is missing or a CUDA device is absent,
every compute entry point raises.  The product path never runs on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
import re

from .errors import STATUS_ERRORS

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SF_LIB_PATH") or os.path.join(_HERE, "libstreamflow.so")  # override: diagnostics
HEADER = os.path.join(os.path.dirname(_HERE), "include", "streamflow.h")

SF_OK = 0
SF_ERR_PARAMETER, SF_ERR_TIME_DOMAIN, SF_ERR_INVARIANT, SF_ERR_STATE, SF_ERR_CUDA = -1, -2, -3, -4, -5
SF_STATUS_TIME_RANGE, SF_STATUS_OFF_GRID, SF_STATUS_DENOM = 1, 2, 4
SF_F32, SF_F64, SF_BF16 = 0, 1, 2
(P_T, P_TNEXT, P_TS, P_TE, P_GAMMA, P_LAMBDA_S, P_ETA_S, P_LAMBDA_T, P_ETA_T,
 P_SPAN, P_DT, P_AT_END) = range(12)
PARAM_STRIDE = 12


class SfSchedule(C.Structure):
    _fields_ = [
        ("boundaries", C.c_void_p), ("abar", C.c_void_p), ("grid", C.c_void_p),
        ("num_windows", C.c_int32), ("t_max", C.c_int32), ("num_steps", C.c_int32),
        ("_pad", C.c_int32), ("eps", C.c_double),
    ]


_vp, _i64, _i32, _f64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double

# name -> argtypes (restype is int unless stated)
SIGNATURES = {
    "sf_version": [],
    "sf_device_sm_count": [],
    "sf_window_params": [C.POINTER(SfSchedule), _vp, _i64, _vp, _vp, _vp],
    "sf_schedule_indices": [C.POINTER(SfSchedule), _vp, _i64, _vp, _vp, _vp, _vp],
    "sf_velocity_step": [_vp, C.c_int, _vp, _vp, C.c_int, _vp, _i64, _i64, _vp],
    "sf_cfg_combine": [_vp, C.c_int, _i64, _i64, _f64, _vp, _vp],
    "sf_mock_keys": [_i64, _vp, _vp, _vp, _i64, _i32, _vp, _vp],
    "sf_mock_eps": [_vp, _i64, _i64, _vp, _vp],
    "sf_stream_prepare": [_vp, _i64, _i32, _i64, _vp, _vp, _vp, _vp],
    "sf_stream_mock_step": [_vp, _i64, _i32, _i64, _i64, C.c_int, _vp, _vp, _vp, _vp, _i64,
                            _vp, _vp, _i32, _f64, _vp, _vp, _vp, _vp, _vp, _vp],
    "sf_stream_reset": [_vp, _i64, _i32, _i64, C.c_int, _vp, _vp, _vp],
    "sf_gemm_bf16": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i32, _vp],
    "sf_gemm_qkv": [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, C.c_float, _vp],
    "sf_gemm_res_ln": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i32,
                       C.c_float, _vp],
    "sf_gemm_qkv_hd": [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, C.c_float, _vp],
    "sf_gemm_res": [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i32, _vp],
    "sf_ln_modulate": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i32, C.c_float, _vp],
    "sf_analytic_eps": [_vp, _vp, _vp, C.c_int, _vp, _i64, _i64, _vp, _vp],
    "sf_attention": [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp],
    "sf_attention_hd": [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp],
    "sf_numpy_normal": [_vp, _i64, _i64, _i64, _vp, C.c_int, _vp],
    "sf_philox_normal": [_vp, _i64, _i64, C.c_uint64, _i64, _vp],
    "sf_block_tail": [_vp] * 15 + [_i64, C.c_float, _i64, _i32, _vp],
}

_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares (``int sf_xxx(`` / ``const char* sf_xxx(``)."""
    with open(HEADER) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sf_\w+)\s*\(", text, re.M)))


RESTYPES = {"sf_version": C.c_char_p, "sf_dit_workspace_bytes": C.c_int64}


def load():
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2511_22009_b200.build` "
            "(there is no CPU fallback)")
    _lib = C.CDLL(LIB_PATH)
    return _lib


def fn(name: str):
    """The library function ``name`` with its ctypes signature applied."""
    f = getattr(load(), name)
    if name not in SIGNATURES:  # ctypes would pass 64-bit pointers / seeds as 32-bit ints
        raise RuntimeError(f"{name}: no ctypes signature registered")
    if f.argtypes is None:
        f.argtypes = SIGNATURES[name]
        f.restype = RESTYPES.get(name, C.c_int)
    return f


_ERRS = STATUS_ERRORS
assert set(_ERRS) == {SF_ERR_PARAMETER, SF_ERR_TIME_DOMAIN, SF_ERR_INVARIANT, SF_ERR_STATE}


def check(code: int, what: str) -> None:
    if code == SF_OK:
        return
    exc = _ERRS.get(code)
    if exc is not None:
        raise exc(f"{what}: rejected by libstreamflow (code {code})")
    raise RuntimeError(f"{what}: CUDA failure in libstreamflow (code {code})")


def call(name: str, *args) -> None:
    check(fn(name)(*args), name)
