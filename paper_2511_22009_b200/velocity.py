"""Heterogeneous-timestep Euler step on the GPU (drop-in for flowpipe velocity.py).

``batched_velocity_step`` keeps the reference signature and semantics
(velocity.py:93-135): a new LatentBatch is returned, inputs are untouched.
It accepts numpy arrays (results come back as numpy, bit-identical to the
reference) or CUDA tensors (results stay on the device).  The arithmetic is
kernel K1 (window coefficients, fp64) + K10-lite (Euler in the latent dtype)
from libstreamflow.so.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ParameterError
from .schedule import DeviceSchedule, TimeWindowSchedule


def _is_torch(a) -> bool:
    return isinstance(a, torch.Tensor)


@dataclass(frozen=True)
class LatentBatch:
    """B latent rows + per-row flow time + generation id (velocity.py:31-57).
    Arrays may be numpy (host) or torch CUDA tensors (device)."""

    data: object
    timesteps: object
    ids: object

    @property
    def batch_size(self) -> int:
        return int(self.data.shape[0])

    @property
    def dim(self) -> int:
        return int(self.data.shape[1])

    def validate(self) -> None:
        if self.data.ndim != 2:
            raise ParameterError(f"data must be 2-D, got shape {tuple(self.data.shape)}")
        b = self.data.shape[0]
        if len(self.timesteps) != b or len(self.ids) != b:
            raise ParameterError(f"row mismatch: {b} latents, {len(self.timesteps)} timesteps, {len(self.ids)} ids")
        ts = self.timesteps
        lo, hi = (ts.min(), ts.max()) if len(ts) else (0.0, 0.0)
        if float(lo) < 0.0 or float(hi) > 1.0:
            raise ParameterError("timesteps must lie in [0, 1]")


def make_latent_batch(data, timesteps, ids) -> LatentBatch:
    """velocity.py:60-69 (numpy inputs -> fp64 / int64, like the reference)."""
    if _is_torch(data):
        b = LatentBatch(data=data, timesteps=torch.as_tensor(timesteps, dtype=torch.float64, device=data.device),
                        ids=torch.as_tensor(ids, dtype=torch.int64, device=data.device))
    else:
        b = LatentBatch(data=np.asarray(data, dtype=np.float64), timesteps=np.asarray(timesteps, dtype=np.float64),
                        ids=np.asarray(ids, dtype=np.int64))
    b.validate()
    return b


@dataclass
class StepStats:
    """velocity.py:72-90."""

    param_evals: int = 0
    elementwise_ops: int = 0
    scheduler_calls: int = field(default=0)

    def merge(self, other: "StepStats") -> None:
        self.param_evals += other.param_evals
        self.elementwise_ops += other.elementwise_ops
        self.scheduler_calls += other.scheduler_calls


_DT = {torch.float32: _lib.SF_F32, torch.float64: _lib.SF_F64}


def _to_device(a, dtype=None) -> torch.Tensor:
    t = a if _is_torch(a) else torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda().contiguous()


def velocity_step_device(eps: torch.Tensor, x: torch.Tensor, params: torch.Tensor,
                         out: torch.Tensor | None = None) -> torch.Tensor:
    """K10-lite on device tensors: x_next = x + dt*(lam x + eta eps - x)/span per row."""
    if x.dtype not in _DT or eps.dtype not in _DT:
        raise ParameterError(f"unsupported dtypes {x.dtype}/{eps.dtype}")
    B, D = x.shape
    if out is None:
        out = torch.empty_like(x)
    _lib.call("sf_velocity_step", eps.data_ptr(), _DT[eps.dtype], x.data_ptr(), out.data_ptr(), _DT[x.dtype],
              params.data_ptr(), B, D, torch.cuda.current_stream().cuda_stream)
    return out


def batched_velocity_step(model_out, batch: LatentBatch, sched: TimeWindowSchedule,
                          stats: StepStats | None = None) -> LatentBatch:
    """velocity.py:93-135 on the GPU.  ParameterError on shape mismatch,
    TimeDomainError for off-grid timesteps (raised before any state changes)."""
    if tuple(model_out.shape) != tuple(batch.data.shape):
        raise ParameterError(f"model output shape {tuple(model_out.shape)} != batch shape {tuple(batch.data.shape)}")
    host = not _is_torch(batch.data)
    x = _to_device(batch.data)
    if x.dtype not in _DT:
        x = x.to(torch.float64)
    ts = _to_device(batch.timesteps, torch.float64)
    e = _to_device(model_out)
    if e.dtype not in _DT:
        e = e.to(torch.float64)
    dev = DeviceSchedule.of(sched)
    params = dev.params(ts)
    x_next = velocity_step_device(e, x, params)
    t_next = params[:, _lib.P_TNEXT].contiguous()
    if stats is not None:
        stats.param_evals += batch.batch_size
        stats.elementwise_ops += 3
        stats.scheduler_calls += 1
    if host:
        return LatentBatch(data=x_next.cpu().numpy(), timesteps=t_next.cpu().numpy(), ids=batch.ids)
    return LatentBatch(data=x_next, timesteps=t_next, ids=batch.ids)


def sequential_velocity_step(model_out, latent, t: float, sched: TimeWindowSchedule,
                             stats: StepStats | None = None):
    """Single-row step (velocity.py:138-181) through the same device kernels."""
    x_row = np.asarray(latent, dtype=np.float64).reshape(1, -1)
    e_row = np.asarray(model_out, dtype=np.float64).reshape(1, -1)
    if x_row.shape != e_row.shape:
        raise ParameterError(f"model output length {e_row.shape[1]} != latent length {x_row.shape[1]}")
    out = batched_velocity_step(e_row, LatentBatch(x_row, np.array([float(t)]), np.array([0])), sched)
    if stats is not None:
        stats.param_evals += 1
        stats.elementwise_ops += 3
        stats.scheduler_calls += 1
    return out.data[0], float(out.timesteps[0])
