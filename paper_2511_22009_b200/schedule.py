"""Scheduler arguments and per-timestep window coefficients.

Construction of the schedule objects is host-side argument plumbing with the
reference's exact signatures and validation (flowpipe schedule.py:33-173): the
alpha-bar table, window boundaries and inference grid are O(t_max) constants
built once.  The per-timestep coefficient math (schedule.py:201-295) runs on
the GPU (``sf_window_params``, kernel K1) and is bit-exact with the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InvariantError, ParameterError, TimeDomainError

DEFAULT_T_MAX = 1000
DEFAULT_BETA_START = 1e-4
DEFAULT_BETA_END = 0.02
DEFAULT_NUM_WINDOWS = 4
DEFAULT_EPS = 1e-6
DEFAULT_INFERENCE_STEPS = 4


@dataclass(frozen=True)
class NoiseSchedule:
    """Linear-beta diffusion table (schedule.py:33-60)."""

    betas: np.ndarray
    alphas_cumprod: np.ndarray
    t_max: int

    def validate(self) -> None:
        if self.t_max < 2:
            raise ParameterError(f"t_max must be >= 2, got {self.t_max}")
        if len(self.betas) != self.t_max or len(self.alphas_cumprod) != self.t_max:
            raise ParameterError("betas and alphas_cumprod must both have length t_max")
        if np.any(self.betas <= 0.0) or np.any(self.betas >= 1.0):
            raise ParameterError("all betas must lie in (0, 1)")
        if np.any(self.alphas_cumprod <= 0.0) or np.any(self.alphas_cumprod > 1.0):
            raise ParameterError("alphas_cumprod must lie in (0, 1]")
        if np.any(np.diff(self.alphas_cumprod) >= 0.0):
            raise ParameterError("alphas_cumprod must be strictly decreasing")


def build_noise_schedule(t_max: int = DEFAULT_T_MAX, beta_start: float = DEFAULT_BETA_START,
                         beta_end: float = DEFAULT_BETA_END) -> NoiseSchedule:
    """schedule.py:63-84."""
    if t_max < 2:
        raise ParameterError(f"t_max must be >= 2, got {t_max}")
    if not (0.0 < beta_start <= beta_end < 1.0):
        raise ParameterError(f"need 0 < beta_start <= beta_end < 1, got ({beta_start}, {beta_end})")
    betas = np.linspace(beta_start, beta_end, t_max, dtype=np.float64)
    ns = NoiseSchedule(betas=betas, alphas_cumprod=np.cumprod(1.0 - betas), t_max=t_max)
    ns.validate()
    return ns


@dataclass(frozen=True)
class TimeWindowSchedule:
    """Window partition + inference grid (schedule.py:87-133)."""

    boundaries: np.ndarray
    eps: float
    noise_schedule: NoiseSchedule
    inference_grid: np.ndarray

    @property
    def num_windows(self) -> int:
        return len(self.boundaries) - 1

    @property
    def num_steps(self) -> int:
        return len(self.inference_grid)

    def validate(self) -> None:
        b = self.boundaries
        if len(b) < 2:
            raise ParameterError("need at least one window (two boundaries)")
        if b[0] != 0.0 or b[-1] != 1.0:
            raise ParameterError("boundaries must start at 0 and end at 1")
        widths = np.diff(b)
        if np.any(widths <= 0.0):
            raise ParameterError("boundaries must be strictly increasing")
        if self.eps <= 0.0:
            raise ParameterError(f"eps must be > 0, got {self.eps}")
        if self.eps >= float(widths.min()) / 2.0:
            raise ParameterError("eps must be smaller than half the narrowest window")
        g = self.inference_grid
        if len(g) < 1:
            raise ParameterError("inference grid must not be empty")
        if np.any(g < 0.0) or np.any(g > 1.0):
            raise ParameterError("inference grid values must lie in [0, 1]")
        if len(g) > 1 and np.any(np.diff(g) <= 0.0):
            raise ParameterError("inference grid must be strictly increasing")


def uniform_inference_grid(num_steps: int) -> np.ndarray:
    """i / num_steps (schedule.py:136-140)."""
    if num_steps < 1:
        raise ParameterError(f"num_steps must be >= 1, got {num_steps}")
    return np.arange(num_steps, dtype=np.float64) / float(num_steps)


def build_time_window_schedule(noise_schedule: NoiseSchedule | None = None,
                               num_windows: int = DEFAULT_NUM_WINDOWS,
                               boundaries=None, eps: float = DEFAULT_EPS,
                               inference_steps: int = DEFAULT_INFERENCE_STEPS,
                               inference_grid=None) -> TimeWindowSchedule:
    """schedule.py:143-173 (same arguments, same validation)."""
    if noise_schedule is None:
        noise_schedule = build_noise_schedule()
    if boundaries is None:
        if num_windows < 1:
            raise ParameterError(f"num_windows must be >= 1, got {num_windows}")
        bounds = np.linspace(0.0, 1.0, num_windows + 1, dtype=np.float64)
    else:
        bounds = np.asarray(boundaries, dtype=np.float64)
    grid = uniform_inference_grid(inference_steps) if inference_grid is None else \
        np.asarray(inference_grid, dtype=np.float64)
    sched = TimeWindowSchedule(boundaries=bounds, eps=eps, noise_schedule=noise_schedule, inference_grid=grid)
    sched.validate()
    return sched


@dataclass(frozen=True)
class WindowParams:
    """Per-sample window coefficients (schedule.py:176-192)."""

    t_s: np.ndarray
    t_e: np.ndarray
    gamma: np.ndarray
    lambda_s: np.ndarray
    eta_s: np.ndarray
    lambda_t: np.ndarray
    eta_t: np.ndarray


class DeviceSchedule:
    """The schedule's fp64 tables resident on the GPU + the C struct that names them."""

    _cache: dict = {}

    def __init__(self, sched: TimeWindowSchedule, device: str = "cuda"):
        self.sched = sched
        self.boundaries = torch.as_tensor(sched.boundaries, dtype=torch.float64).to(device)
        self.abar = torch.as_tensor(sched.noise_schedule.alphas_cumprod, dtype=torch.float64).to(device)
        self.grid = torch.as_tensor(sched.inference_grid, dtype=torch.float64).to(device)
        self.struct = _lib.SfSchedule(self.boundaries.data_ptr(), self.abar.data_ptr(), self.grid.data_ptr(),
                                      sched.num_windows, sched.noise_schedule.t_max, sched.num_steps, 0,
                                      float(sched.eps))
        self.status = torch.zeros(1, dtype=torch.int32, device=device)

    @classmethod
    def of(cls, sched: TimeWindowSchedule) -> "DeviceSchedule":
        key = id(sched)
        hit = cls._cache.get(key)
        if hit is None or hit.sched is not sched:
            hit = cls(sched)
            cls._cache[key] = hit
        return hit

    def params(self, ts: torch.Tensor, out: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
        """K1 over device flow times -> [B, 12] fp64 coefficients; raises the
        reference's exception on off-grid / out-of-range t or a bad denominator."""
        ts = ts.to(dtype=torch.float64).contiguous()
        B = ts.numel()
        if out is None:
            out = torch.empty(B, _lib.PARAM_STRIDE, dtype=torch.float64, device=ts.device)
        self.status.zero_()
        _lib.call("sf_window_params", C.byref(self.struct), ts.data_ptr(), B, out.data_ptr(),
                  self.status.data_ptr(), torch.cuda.current_stream().cuda_stream)
        if check:
            st = int(self.status.item())
            if st & _lib.SF_STATUS_TIME_RANGE:
                raise TimeDomainError(f"timesteps outside [0, 1]: {ts[:4].tolist()}")
            if st & _lib.SF_STATUS_DENOM:
                raise InvariantError("window parameter denominator is non-positive")
            if st & _lib.SF_STATUS_OFF_GRID:
                raise TimeDomainError("timesteps not on the inference grid")
        return out


def _device_ts(ts) -> torch.Tensor:
    return torch.as_tensor(np.asarray(ts, dtype=np.float64).reshape(-1)).cuda()


def window_params(ts, sched: TimeWindowSchedule) -> WindowParams:
    """schedule.py:224-263 on the GPU (no grid-membership requirement)."""
    dev = DeviceSchedule.of(sched)
    t = _device_ts(ts)
    out = dev.params(t, check=False)
    st = int(dev.status.item())
    if st & _lib.SF_STATUS_TIME_RANGE:
        raise TimeDomainError(f"timesteps outside [0, 1]: {np.asarray(ts).reshape(-1)[:4]}")
    if st & _lib.SF_STATUS_DENOM:
        raise InvariantError("window parameter denominator is non-positive")
    o = out.cpu().numpy()
    return WindowParams(t_s=o[:, _lib.P_TS], t_e=o[:, _lib.P_TE], gamma=o[:, _lib.P_GAMMA],
                        lambda_s=o[:, _lib.P_LAMBDA_S], eta_s=o[:, _lib.P_ETA_S],
                        lambda_t=o[:, _lib.P_LAMBDA_T], eta_t=o[:, _lib.P_ETA_T])


def alpha_bar_index(ts, t_max: int) -> np.ndarray:
    """Noise-table index per flow time, round half up, clamped (schedule.py:201-205), on
    the GPU with the same fp64 operation order the window kernel uses."""
    t = _device_ts(ts)
    out = torch.empty(t.numel(), dtype=torch.int64, device=t.device)
    s = _lib.SfSchedule(None, None, None, 0, int(t_max), 0, 0, 0.0)
    _lib.call("sf_schedule_indices", C.byref(s), t.data_ptr(), t.numel(), out.data_ptr(), None, None,
              torch.cuda.current_stream().cuda_stream)
    return out.cpu().numpy()


def grid_indices(ts, sched: TimeWindowSchedule) -> np.ndarray:
    """Inference-grid index per t within eps (schedule.py:266-284); TimeDomainError when
    a t is out of [0, 1] or off the grid."""
    dev = DeviceSchedule.of(sched)
    t = _device_ts(ts)
    out = torch.empty(t.numel(), dtype=torch.int64, device=t.device)
    dev.status.zero_()
    _lib.call("sf_schedule_indices", C.byref(dev.struct), t.data_ptr(), t.numel(), None, out.data_ptr(),
              dev.status.data_ptr(), torch.cuda.current_stream().cuda_stream)
    st = int(dev.status.item())
    if st & _lib.SF_STATUS_TIME_RANGE:
        raise TimeDomainError(f"timesteps outside [0, 1]: {np.asarray(ts).reshape(-1)[:4]}")
    if st & _lib.SF_STATUS_OFF_GRID:
        raise TimeDomainError("timesteps not on the inference grid")
    return out.cpu().numpy()


def window_lookup(ts, sched: TimeWindowSchedule) -> np.ndarray:
    """Window index per t (schedule.py:208-221), derived from the device t_s."""
    wp = window_params(ts, sched)
    return np.searchsorted(sched.boundaries, wp.t_s).astype(np.int64)


def next_timestep(ts, sched: TimeWindowSchedule) -> np.ndarray:
    """Grid successor (schedule.py:287-295) on the GPU; TimeDomainError off-grid."""
    out = DeviceSchedule.of(sched).params(_device_ts(ts))
    return out[:, _lib.P_TNEXT].cpu().numpy()
