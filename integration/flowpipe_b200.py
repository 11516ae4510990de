"""Reference-side binding: what a flowpipe maintainer adds to the
reference package to forward its hot path -- the heterogeneous-timestep Euler step,
flowpipe/velocity.py:93-135 -- to libstreamflow.so through ctypes, with nothing from this
repository's Python package.  Device memory comes from torch; the C ABI is
include/streamflow.h (sf_window_params, sf_velocity_step).

    import flowpipe; from integration import flowpipe_b200 as b200
    b200.install(flowpipe, "/path/to/libstreamflow.so")   # flowpipe.run_stream now steps on the GPU

tests/test_gpu_integration.py runs it against the unmodified reference installed in
baseline/_ref and checks the results bit for bit against the reference's own numpy step.
"""

import ctypes as C

import numpy as np
import torch

F32, F64 = 0, 1              # SF_F32 / SF_F64
STRIDE, P_TNEXT = 12, 1      # SF_PARAM_STRIDE, SF_P_TNEXT
TIME_RANGE, OFF_GRID, DENOM = 1, 2, 4  # SF_STATUS_*


class SfSchedule(C.Structure):  # sf_schedule
    _fields_ = [("boundaries", C.c_void_p), ("abar", C.c_void_p), ("grid", C.c_void_p),
                ("num_windows", C.c_int32), ("t_max", C.c_int32), ("num_steps", C.c_int32),
                ("_pad", C.c_int32), ("eps", C.c_double)]


def install(flowpipe, lib_path):
    """Replace flowpipe.velocity.batched_velocity_step (and the pipeline's reference to it) by
    the library's kernels; returns the new function."""
    sf = C.CDLL(lib_path)
    sf.sf_window_params.argtypes = [C.POINTER(SfSchedule), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                    C.c_void_p]
    sf.sf_velocity_step.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
                                    C.c_int64, C.c_void_p]
    errors, velocity = flowpipe.errors, flowpipe.velocity

    def dev(a, dtype):
        return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)

    def batched_velocity_step(model_out, batch, sched, stats=None):
        eps = np.asarray(model_out)
        if eps.shape != batch.data.shape:  # velocity.py:110-113
            raise errors.ParameterError(f"model output shape {eps.shape} != batch shape {batch.data.shape}")
        xdt = torch.float32 if batch.data.dtype == np.float32 else torch.float64
        edt = torch.float32 if eps.dtype == np.float32 else torch.float64
        x, e = dev(batch.data, xdt), dev(eps, edt)
        ts = dev(batch.timesteps, torch.float64)
        tables = [dev(sched.boundaries, torch.float64), dev(sched.noise_schedule.alphas_cumprod, torch.float64),
                  dev(sched.inference_grid, torch.float64)]
        s = SfSchedule(*[t.data_ptr() for t in tables], sched.num_windows, sched.noise_schedule.t_max,
                       sched.num_steps, 0, sched.eps)
        B, D = x.shape
        params = torch.empty(B, STRIDE, dtype=torch.float64, device="cuda")
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        stream = torch.cuda.current_stream().cuda_stream
        if sf.sf_window_params(C.byref(s), ts.data_ptr(), B, params.data_ptr(), status.data_ptr(), stream) != 0:
            raise RuntimeError("sf_window_params failed")
        st = int(status.item())
        if st & TIME_RANGE:
            raise errors.TimeDomainError(f"timesteps outside [0, 1]: {batch.timesteps[:4]}")
        if st & DENOM:
            raise errors.InvariantError("window parameter denominator is non-positive")
        if st & OFF_GRID:
            raise errors.TimeDomainError(f"timesteps not on the inference grid: {batch.timesteps[:4]}")
        out = torch.empty_like(x)
        if sf.sf_velocity_step(e.data_ptr(), F64 if edt == torch.float64 else F32, x.data_ptr(), out.data_ptr(),
                               F64 if xdt == torch.float64 else F32, params.data_ptr(), B, D, stream) != 0:
            raise RuntimeError("sf_velocity_step failed")
        if stats is not None:  # velocity.py:131-134
            stats.param_evals += B
            stats.elementwise_ops += 3
            stats.scheduler_calls += 1
        return velocity.LatentBatch(data=out.cpu().numpy(), timesteps=params[:, P_TNEXT].cpu().numpy(),
                                    ids=batch.ids)

    velocity.batched_velocity_step = batched_velocity_step
    flowpipe.pipeline.batched_velocity_step = batched_velocity_step
    flowpipe.batched_velocity_step = batched_velocity_step
    return batched_velocity_step
