"""Stream batch (Alg. 2) with a device-resident ring buffer.

Drop-in for flowpipe pipeline.py:139-266 (``run_stream``, ``run_vanilla`` and
their result / stats types) plus the device-resident ``StreamBatch`` the
north star asks for: S independent streams x n in-flight slots, advanced in
lockstep, one velocity evaluation per iteration for every slot.

Ring layout: row r = s*n + k holds generation g of stream s
with g = k (mod n); at iteration j its stage is (j - k) mod n and it is active
iff 0 <= g < m.  The reference's ``buffer.insert(0, ...)`` / ``pop()`` shift is
the implicit advance of j -- nothing moves in memory; the slot that retires
generation j-n+1 is refilled in the same kernel with the noise of generation
j+1.  Everything between ``step()`` calls stays on the GPU.
"""

from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _lib
from .errors import ParameterError, StateError
from .engine import model_forward
from .models import (Conditioning, DiTVelocityModel, SeededMockModel, VelocityModel, apply_cfg, busy_wait_us,
                     handle_cfg)
from .schedule import DeviceSchedule, TimeWindowSchedule
from .velocity import LatentBatch, StepStats, batched_velocity_step, sequential_velocity_step, velocity_step_device


# ----------------------------------------------------------------------------- reference result / stats types
@dataclass
class BufferEntry:
    """pipeline.py:31-37."""

    latent: np.ndarray
    gen_id: int
    stage: int


@dataclass
class PipelineState:
    """Newest-first snapshot (pipeline.py:40-50)."""

    buffer: list
    stage_times: np.ndarray
    emitted: int
    iteration: int


@dataclass(frozen=True)
class DecodedPayload:
    """decode_stub's payload (pipeline.py:53-56); ``image`` is set when a device
    decoder (vae.TinyDecoder) decoded the frame: [3, 512, 512] fp32."""

    latent: np.ndarray
    image: np.ndarray | None = None


@dataclass(frozen=True)
class GenerationResult:
    id: int
    latent: np.ndarray
    decoded: DecodedPayload
    iterations_spanned: int


@dataclass
class RunStats:
    """pipeline.py:68-83."""

    model_calls: int = 0
    scheduler_calls: int = 0
    decodes: int = 0
    decode_time_us: float = 0.0
    step_stats: StepStats = field(default_factory=StepStats)

    def merge(self, other: "RunStats") -> None:
        self.model_calls += other.model_calls
        self.scheduler_calls += other.scheduler_calls
        self.decodes += other.decodes
        self.decode_time_us += other.decode_time_us
        self.step_stats.merge(other.step_stats)


def decode_stub(latent, cost_us: float = 0.0) -> DecodedPayload:
    """Identity decode with injected cost (pipeline.py:86-89)."""
    busy_wait_us(cost_us)
    return DecodedPayload(latent=np.array(latent, copy=True))


def generation_noise(seed: int, gen_id: int, dim: int) -> np.ndarray:
    """Initial noise of one generation (pipeline.py:92-98): numpy PCG64 seeded
    by [seed, id].  This is the *input* of a generation; the device ring ingests
    it (parity mode) or replaces it with on-device Philox (throughput mode)."""
    return np.random.default_rng([seed, gen_id]).standard_normal(dim)


def numpy_noise_device(seeds, gen: int, dim: int, dtype=torch.float64, out: torch.Tensor | None = None,
                       device: str = "cuda") -> torch.Tensor:
    """generation_noise for every seed at once, on the device: row s of the result is
    bit-identical to ``np.random.default_rng([seeds[s], gen]).standard_normal(dim)``
    (cast to fp32 with round-to-nearest when dtype is float32, as pipeline.py:176 does).
    sf_numpy_normal: SeedSequence -> PCG64 -> numpy's ziggurat on the GPU."""
    if isinstance(seeds, torch.Tensor) and seeds.is_cuda:
        sd = seeds.to(torch.int64).contiguous()
    else:
        vals = [int(v) for v in (seeds if isinstance(seeds, (list, tuple)) else np.asarray(seeds).ravel())]
        if any(v < 0 for v in vals) or gen < 0:
            raise ValueError("expected non-negative integer")  # numpy's SeedSequence error
        if any(v >= 1 << 63 for v in vals):
            raise ParameterError("seeds must be < 2**63 for the device generator")
        sd = torch.tensor(vals, dtype=torch.int64, device=device)
    S = sd.numel()
    if out is None:
        out = torch.empty(S, dim, dtype=dtype, device=sd.device)
    if out.shape != (S, dim) or not out.is_contiguous() or out.dtype not in (torch.float32, torch.float64):
        raise ParameterError("out must be a contiguous [S, dim] float32/float64 tensor")
    _lib.call("sf_numpy_normal", sd.data_ptr(), int(gen), S, int(dim), out.data_ptr(),
              _lib.SF_F64 if out.dtype == torch.float64 else _lib.SF_F32, torch.cuda.current_stream().cuda_stream)
    return out


def _check_run_args(m: int, n: int, sched: TimeWindowSchedule) -> None:
    if m < 1:
        raise ParameterError(f"need at least one generation, got m={m}")
    if n < 1:
        raise ParameterError(f"need at least one denoising step, got n={n}")
    if sched.num_steps < n:
        raise ParameterError(f"inference grid has {sched.num_steps} points, fewer than n={n} steps")


_UNBOUNDED = 1 << 62


class StreamBatch:
    """Device-resident heterogeneous-timestep stream batch.

    model      SeededMockModel / DiTVelocityModel (fused native step) or any
               VelocityModel (generic path: model.forward + device Euler)
    sched      TimeWindowSchedule (reference scheduler / time-grid arguments)
    n          steps per generation (= in-flight slots per stream)
    num_streams S independent streams (own seed and conditioning each)
    cond       one Conditioning for all streams or a list of S
    seed       run seed of stream 0 (stream s uses seed + s) or a list of S
    m          generations per stream (None = unbounded serving)
    dtype      latent dtype (np.float64 / np.float32; the DiT keeps fp32)
    noise      "numpy": generation_noise bit-identical to the reference, drawn on
                        the device (sf_numpy_normal: SeedSequence/PCG64/ziggurat),
               "numpy_host": the same noise computed by numpy on the host and
                        uploaded (cross-check path),
               "device": on-device Philox N(0,1) (throughput mode),
               "host":  caller-provided noise via launch_host_io
    """

    def __init__(self, model: VelocityModel, sched: TimeWindowSchedule, n: int, num_streams: int = 1,
                 cond: Conditioning | list | None = None, seed: int | list = 0, m: int | None = None,
                 dtype=np.float64, noise: str = "numpy", use_graph: bool = True, device: str = "cuda",
                 decoder=None):
        if not torch.cuda.is_available():
            raise RuntimeError("StreamBatch needs a CUDA device; there is no CPU fallback")
        _check_run_args(1 if m is None else m, n, sched)
        if num_streams < 1:
            raise ParameterError(f"need at least one stream, got {num_streams}")
        if noise not in ("numpy", "numpy_host", "device", "host"):
            raise ParameterError(f"noise must be 'numpy', 'numpy_host', 'device' or 'host', got {noise!r}")
        self.model, self.sched, self.n, self.S = model, sched, int(n), int(num_streams)
        self.m = _UNBOUNDED if m is None else int(m)
        self.noise, self.use_graph, self.device = noise, bool(use_graph), device
        self.D = model.dim
        self.kind = ("dit" if isinstance(model, DiTVelocityModel) else
                     "mock" if isinstance(model, SeededMockModel) else "generic")
        self.np_dtype = np.dtype(dtype)
        if self.np_dtype not in (np.float32, np.float64):
            raise ParameterError(f"unsupported latent dtype {dtype}")
        if self.kind == "dit" and self.np_dtype != np.float32:
            raise ParameterError("the DiT stream batch keeps fp32 latents; pass dtype=np.float32")
        self.t_dtype = torch.float64 if self.np_dtype == np.float64 else torch.float32
        conds = cond if isinstance(cond, (list, tuple)) else [cond] * self.S
        if len(conds) != self.S or any(c is None for c in conds):
            raise ParameterError("need one Conditioning (or a list of num_streams)")
        # guidance per stream (independent run_stream calls may differ): the batch is doubled when any
        # stream is guided; the fused kernels combine with each stream's own w (w == 1: unguided)
        scales = [float(c.guidance_scale) for c in conds]
        guided = [w for w in scales if w != 1.0]
        self.w = guided[0] if guided else 1.0
        self.w_streams = (torch.tensor(scales, dtype=torch.float64, device=device)
                          if len(set(scales)) > 1 else None)
        self.conds = conds
        self.seeds = list(seed) if isinstance(seed, (list, tuple)) else [int(seed) + s for s in range(self.S)]
        E = model.embed_dim
        for c in conds:
            if c.embed_dim != E:
                raise ParameterError(f"embedding length {c.embed_dim} != model embed_dim {E}")
        dev = device
        R = self.S * self.n
        if self.kind == "dit" and (2 if self.w != 1.0 else 1) * R > model.max_rows:
            raise ParameterError(f"{R} slots (x2 with CFG) exceed the model's max_rows {model.max_rows}")
        self.dsched = DeviceSchedule.of(sched)
        self.stage_params = self.dsched.params(self.dsched.grid[: self.n].clone()).contiguous()
        self.stage_times = np.asarray(sched.inference_grid[: self.n], dtype=np.float64).copy()
        self.ctl = torch.zeros(4, dtype=torch.int64, device=dev)
        self.row_info = torch.zeros(R * 4, dtype=torch.int64, device=dev)
        self.row_t = torch.zeros(R, dtype=torch.float64, device=dev)
        self.x_ring = torch.zeros(R, self.D, dtype=self.t_dtype, device=dev)
        self.frames = torch.zeros(self.S, self.D, dtype=self.t_dtype, device=dev)
        self.frame_ids = torch.full((self.S,), -1, dtype=torch.int64, device=dev)
        self.emb = torch.as_tensor(np.stack([c.embedding for c in conds]), dtype=torch.float64).to(dev).contiguous()
        negs = [c.negative_embedding for c in conds]
        self.neg = None if all(x is None for x in negs) else torch.as_tensor(
            np.stack([np.zeros(E) if x is None else x for x in negs]), dtype=torch.float64).to(dev).contiguous()
        noise_dt = torch.float32 if self.kind == "dit" else torch.float64
        self.noise_dev = torch.zeros(self.S, self.D, dtype=noise_dt, device=dev)
        self.noise_host = torch.zeros(self.S, self.D, dtype=noise_dt).pin_memory() if noise == "numpy_host" else None
        self.noise_seed = int(self.seeds[0]) & ((1 << 64) - 1)
        if noise in ("device", "host") and any(int(v) != int(self.seeds[0]) + s for s, v in enumerate(self.seeds)):
            # the Philox generator of stream s is keyed by seeds[0] + s
            raise ParameterError("noise='device'/'host' keys stream s's Philox noise by seeds[0] + s; "
                                 "pass consecutive seeds (or noise='numpy' for arbitrary per-stream seeds)")
        if noise == "numpy":
            if any(int(v) < 0 for v in self.seeds):
                raise ValueError("expected non-negative integer")  # numpy's SeedSequence error
            if any(int(v) >= 1 << 63 for v in self.seeds):
                raise ParameterError("seeds must be < 2**63 for the device generator")
            self.seeds_dev = torch.tensor([int(v) for v in self.seeds], dtype=torch.int64, device=dev)
        self.decoder = decoder
        self.images = None
        if decoder is not None:
            if self.D != 16384 or decoder.max_frames < self.S:
                raise ParameterError("the TAESD decoder takes 4x64x64 latents, one per stream (max_frames >= S)")
            self.images = torch.zeros(self.S, 3, 512, 512, dtype=torch.float32, device=dev)
        self._h2d_done = torch.cuda.Event()
        self._io = None  # launch_host_io's copy streams, events and double buffers (created on first use)
        # the mock step's per-row blake2b keys (cond / uncond), device scratch
        self.mock_keys = torch.empty(2 * R, dtype=torch.int64, device=dev) if self.kind == "mock" else None
        self.stats = [RunStats() for _ in range(self.S)]
        self.j = 0
        self._stream = lambda: torch.cuda.current_stream().cuda_stream
        self.reset()

    def __del__(self):
        # drop the CUDA graphs captured over this batch's buffers before they are freed
        if getattr(self, "kind", None) == "dit" and getattr(self, "use_graph", False):
            try:
                h = self.model.device_model.handle
                if h.value:  # NULL once the model's runtime handle is destroyed (graphs went with it)
                    _lib.fn("sf_dit_graph_release")(h, self.ctl.data_ptr())
            except Exception:
                pass

    def _wptr(self):
        return None if self.w_streams is None else self.w_streams.data_ptr()

    # ------------------------------------------------------------------ admission noise
    def _fill_noise(self, gen: int) -> bool:
        """Stage generation `gen`'s initial noise for every stream; False if none."""
        if gen >= self.m:
            return False
        if self.noise == "numpy":
            numpy_noise_device(self.seeds_dev, gen, self.D, out=self.noise_dev)
        elif self.noise == "numpy_host":
            arr = np.stack([generation_noise(sd, gen, self.D) for sd in self.seeds])
            self._h2d_done.synchronize()  # the previous async copy has left the pinned buffer
            self.noise_host.copy_(torch.from_numpy(arr.astype(self.noise_host.numpy().dtype, copy=False)))
            self.noise_dev.copy_(self.noise_host, non_blocking=True)
            self._h2d_done.record()
        return True

    def reset(self) -> None:
        st = self._stream()
        self.j = 0
        self.stats = [RunStats() for _ in range(self.S)]
        self._fill_noise(0)
        use_host = self.noise in ("numpy", "numpy_host")
        if self.kind == "dit":
            _lib.call("sf_dit_stream_reset", self.ctl.data_ptr(), self.S, self.n, self.D, self.x_ring.data_ptr(),
                      self.noise_dev.data_ptr() if use_host else None, self.noise_seed, st)
        else:
            if not use_host:
                tmp = torch.empty(self.S, self.D, dtype=torch.float32, device=self.device)
                _lib.call("sf_philox_normal", tmp.data_ptr(), self.S, self.D, self.noise_seed, 0, st)
                self.noise_dev.copy_(tmp)
            _lib.call("sf_stream_reset", self.ctl.data_ptr(), self.S, self.n, self.D,
                      _lib.SF_F64 if self.t_dtype == torch.float64 else _lib.SF_F32, self.x_ring.data_ptr(),
                      self.noise_dev.data_ptr(), st)

    @property
    def total_iterations(self) -> int:
        return self.m + self.n - 1

    def done(self) -> bool:
        return self.j >= self.total_iterations

    # ------------------------------------------------------------------ one iteration
    def launch(self) -> int:
        """Enqueue iteration j on the current CUDA stream without any host sync.
        Returns the generation id retiring this iteration (or -1)."""
        if self.done():
            raise StateError("stream batch already drained all generations")
        j, n, m, st = self.j, self.n, self.m, self._stream()
        if self.kind != "generic":
            # the fused step is the iteration's one guided forward: charge the model's declared
            # cost once, as VelocityModel.forward does (models.py:111-114)
            busy_wait_us(self.model.cost_us)
        admit_next = self._fill_noise(j + 1) if self.noise in ("numpy", "numpy_host") else (j + 1 < m)
        if self.kind == "dit":
            _lib.call("sf_dit_stream_step", self.model.device_model.handle, self.ctl.data_ptr(), self.S, n, m,
                      self.stage_params.data_ptr(), self.row_info.data_ptr(), self.row_t.data_ptr(),
                      self.x_ring.data_ptr(), self.emb.data_ptr(), None if self.neg is None else self.neg.data_ptr(),
                      self.w, self._wptr(), self.noise_dev.data_ptr() if self.noise != "device" else None,
                      self.noise_seed, self.frames.data_ptr(), self.frame_ids.data_ptr(), 1 if self.use_graph else 0, st)
        else:
            if self.noise == "device" and admit_next:
                tmp = torch.empty(self.S, self.D, dtype=torch.float32, device=self.device)
                _lib.call("sf_philox_normal", tmp.data_ptr(), self.S, self.D, self.noise_seed, j + 1, st)
                self.noise_dev.copy_(tmp)
            _lib.call("sf_stream_prepare", self.ctl.data_ptr(), self.S, n, m, self.stage_params.data_ptr(),
                      self.row_info.data_ptr(), self.row_t.data_ptr(), st)
            if self.kind == "mock":
                _lib.call("sf_stream_mock_step", self.ctl.data_ptr(), self.S, n, m, self.D,
                          _lib.SF_F64 if self.t_dtype == torch.float64 else _lib.SF_F32, self.x_ring.data_ptr(),
                          self.stage_params.data_ptr(), self.row_info.data_ptr(), self.row_t.data_ptr(),
                          self.model.seed, self.emb.data_ptr(), None if self.neg is None else self.neg.data_ptr(),
                          self.model.embed_dim, self.w, self._wptr(), self.noise_dev.data_ptr(),
                          self.frames.data_ptr(), self.frame_ids.data_ptr(), self.mock_keys.data_ptr(), st)
            else:
                self._generic_step(j)
        lo, hi = max(0, j - n + 1), min(j, m - 1)
        for s in range(self.S):
            rs = self.stats[s]
            rs.model_calls += 1
            rs.scheduler_calls += 1
            rs.step_stats.param_evals += hi - lo + 1
            rs.step_stats.elementwise_ops += 3
            rs.step_stats.scheduler_calls += 1
        self.j += 1
        retiring = j - n + 1
        if 0 <= retiring < m:
            for rs in self.stats:
                rs.decodes += 1
            if self.decoder is not None:  # decode the retired frames on the same stream
                lat = self.frames if self.frames.dtype == torch.float32 else self.frames.float()
                self.decoder.decode(lat.view(self.S, 4, 64, 64), self.images)
            return retiring
        return -1

    def _generic_step(self, j: int) -> None:
        """Any VelocityModel: gather the active rows (newest first), one guided
        forward, device Euler, scatter back, emit, refill."""
        n, m = self.n, self.m
        lo, hi = max(0, j - n + 1), min(j, m - 1)
        gens = list(range(hi, lo - 1, -1))
        rows = [s * n + g % n for s in range(self.S) for g in gens]
        idx = torch.tensor(rows, device=self.device)
        stages = torch.tensor([j - g for _ in range(self.S) for g in gens], device=self.device)
        x = self.x_ring.index_select(0, idx)
        ts = self.dsched.grid.index_select(0, stages)
        ids = torch.tensor([g for _ in range(self.S) for g in gens], device=self.device)
        eps_rows = []
        per = len(gens)
        for s, c in enumerate(self.conds):
            b = LatentBatch(data=x[s * per:(s + 1) * per], timesteps=ts[s * per:(s + 1) * per],
                            ids=ids[s * per:(s + 1) * per])
            if c.guidance_scale != 1.0:
                d2, c2 = apply_cfg(b, c)
                out = handle_cfg(model_forward(self.model, d2, c2), c.guidance_scale)
            else:
                out = model_forward(self.model, b, c)
            e = out.epsilon if isinstance(out.epsilon, torch.Tensor) else torch.from_numpy(out.epsilon).cuda()
            eps_rows.append(e.to(self.x_ring.dtype) if e.dtype not in (torch.float32, torch.float64) else e)
        eps = torch.cat(eps_rows)
        params = self.stage_params.index_select(0, stages).contiguous()
        x_new = velocity_step_device(eps.contiguous(), x.contiguous(), params)
        self.x_ring.index_copy_(0, idx, x_new)
        retiring = j - n + 1
        if 0 <= retiring < m:
            for s in range(self.S):
                self.frames[s].copy_(self.x_ring[s * n + retiring % n])
            self.frame_ids.fill_(retiring)
        else:
            self.frame_ids.fill_(-1)
        if j + 1 < m:
            k = (j + 1) % n
            for s in range(self.S):
                self.x_ring[s * n + k].copy_(self.noise_dev[s].to(self.x_ring.dtype))

    def launch_host_io(self, noise_src: torch.Tensor, frames_dst: torch.Tensor) -> int:
        """End-to-end serving step with HOST buffers (noise="host"): async H2D of
        the admitted generation's noise from pinned ``noise_src`` [S, D], the
        device step, async D2H of the emitted frames into pinned ``frames_dst``;
        no host sync.  The copies run on two side streams (H2D, D2H) against double-buffered
        device noise / frame buffers, so step j's D2H and step j+1's H2D overlap
        the neighbouring steps' kernels (events order each buffer's reuse); call
        ``io_join()`` to make the current stream wait for the outstanding copies.
        ``sb.frames`` is the buffer the latest step wrote (rows of streams that retired no frame
        this step, ``frame_ids == -1``, are stale, as with launch())."""
        if self.noise != "host":
            raise ParameterError("launch_host_io needs a StreamBatch built with noise='host'")
        cur = torch.cuda.current_stream()
        if self._io is None:
            ev = lambda: [torch.cuda.Event(), torch.cuda.Event()]
            self._io = {"cs": torch.cuda.Stream(device=self.device), "cs_out": torch.cuda.Stream(device=self.device),
                        "slot": 0,
                        "noise": [self.noise_dev, torch.empty_like(self.noise_dev)],
                        "frames": [self.frames, torch.zeros_like(self.frames)],
                        "h2d": ev(), "step": ev(), "d2h": ev(), "used": [False, False]}
        io = self._io
        b, cs = io["slot"], io["cs"]
        io["slot"] ^= 1
        with torch.cuda.stream(cs):
            if io["used"][b]:
                cs.wait_event(io["step"][b])  # the step that read noise[b] two steps ago is done
            io["noise"][b].copy_(noise_src, non_blocking=True)
            io["h2d"][b].record(cs)
        cur.wait_event(io["h2d"][b])
        if io["used"][b]:
            cur.wait_event(io["d2h"][b])  # frames[b]'s previous D2H has read it
        self.noise_dev, self.frames = io["noise"][b], io["frames"][b]
        g = self.launch()
        io["step"][b].record(cur)
        co = io["cs_out"]  # D2H on its own stream: it overlaps the next step's H2D (full-duplex link)
        with torch.cuda.stream(co):
            co.wait_event(io["step"][b])
            frames_dst.copy_(io["frames"][b], non_blocking=True)
            io["d2h"][b].record(co)
        io["used"][b] = True
        return g

    def io_join(self) -> None:
        """Make the current stream wait for launch_host_io's outstanding copies."""
        if self._io is not None:
            torch.cuda.current_stream().wait_stream(self._io["cs"])
            torch.cuda.current_stream().wait_stream(self._io["cs_out"])

    def profile_step(self) -> dict:
        """One eager DiT step with a CUDA event after every launch: per kernel
        class {name: (total_ms, launches)} (sf_dit_profile_step)."""
        if self.kind != "dit":
            raise StateError("profile_step is implemented for the DiT stream batch")
        from .dit import PROFILE_CLASSES

        ms = (C.c_float * 16)()
        cnt = (C.c_int32 * 16)()
        j = self.j
        _lib.call("sf_dit_profile_step", self.model.device_model.handle, self.ctl.data_ptr(), self.S, self.n, self.m,
                  self.stage_params.data_ptr(), self.row_info.data_ptr(), self.row_t.data_ptr(),
                  self.x_ring.data_ptr(), self.emb.data_ptr(), None if self.neg is None else self.neg.data_ptr(),
                  self.w, self._wptr(), self.noise_dev.data_ptr() if self.noise != "device" else None,
                  self.noise_seed, self.frames.data_ptr(), self.frame_ids.data_ptr(), ms, cnt, self._stream())
        self.j = j + 1
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(PROFILE_CLASSES)}

    def step(self, decode_cost_us: float = 0.0) -> list:
        """One iteration; returns [(stream, GenerationResult)] for the frames that
        retired (one per stream after warm-up), copied to the host."""
        g = self.launch()
        if g < 0:
            return []
        frames = self.frames.cpu().numpy()
        images = self.images.cpu().numpy() if self.decoder is not None else None
        out = []
        for s in range(self.S):
            lat = frames[s].copy()
            self.stats[s].decode_time_us += decode_cost_us
            dec = decode_stub(lat, decode_cost_us)
            if images is not None:
                dec = DecodedPayload(latent=dec.latent, image=images[s].copy())
            out.append((s, GenerationResult(id=g, latent=lat, decoded=dec, iterations_spanned=self.n)))
        return out

    def __call__(self, m: int | None = None) -> list:
        """Run to completion (m generations per stream); results per stream in
        completion order."""
        if m is not None and m != self.m:
            _check_run_args(m, self.n, self.sched)
            self.m = int(m)
            self.reset()
        if self.m == _UNBOUNDED:
            raise ParameterError("an unbounded StreamBatch has no completion; call step()")
        res = [[] for _ in range(self.S)]
        while not self.done():
            for s, r in self.step():
                res[s].append(r)
        return res

    def snapshot(self, emitted: int) -> PipelineState:
        """Newest-first buffer of stream 0 after the last iteration (pipeline.py:208-219)."""
        j = self.j - 1
        n, m = self.n, self.m
        lo, hi = max(0, j - n + 1), min(j, m - 1)
        ring = self.x_ring[:n].cpu().numpy()
        buf = []
        for g in range(hi, lo - 1, -1):
            stage = j - g + 1
            if stage >= n:
                continue
            buf.append(BufferEntry(latent=ring[g % n].copy(), gen_id=g, stage=stage))
        return PipelineState(buffer=buf, stage_times=self.stage_times, emitted=emitted, iteration=j)


# ----------------------------------------------------------------------------- reference entry points
def run_stream(m: int, n: int, model: VelocityModel, cond: Conditioning, seed: int, sched: TimeWindowSchedule,
               sched_cost_us: float = 0.0, decode_cost_us: float = 0.0, dtype=np.float64,
               on_iteration: Callable[[PipelineState], None] | None = None, decoder=None):
    """pipeline.py:139-220: m generations of n steps in m+n-1 iterations,
    through the device-resident stream batch (one stream).  ``decoder`` (an
    extension: vae.TinyDecoder) decodes each retired frame on the device."""
    _check_run_args(m, n, sched)
    if isinstance(model, DiTVelocityModel) and np.dtype(dtype) == np.float64:
        # the reference's default latent dtype is fp64; the DiT ring is fp32 (bf16 network): say so
        warnings.warn("run_stream: the DiT velocity field keeps fp32 latents; dtype=float64 runs as float32",
                      RuntimeWarning, stacklevel=2)
        dtype = np.float32
    sb = StreamBatch(model, sched, n, num_streams=1, cond=cond, seed=seed, m=m, dtype=dtype, noise="numpy",
                     decoder=decoder)
    results = []
    while not sb.done():
        busy_wait_us(sched_cost_us)
        for _, r in sb.step(decode_cost_us):
            results.append(r)
        if on_iteration is not None:
            on_iteration(sb.snapshot(len(results)))
    return results, sb.stats[0]


def run_vanilla(m: int, n: int, model: VelocityModel, cond: Conditioning, seed: int, sched: TimeWindowSchedule,
                sched_cost_us: float = 0.0, decode_cost_us: float = 0.0):
    """pipeline.py:223-266: one generation at a time, m*n single-row calls."""
    _check_run_args(m, n, sched)
    stats = RunStats()
    results = []
    for g in range(m):
        latent = generation_noise(seed, g, model.dim)
        t = float(sched.inference_grid[0])
        for _ in range(n):
            batch = LatentBatch(data=latent[None, :], timesteps=np.asarray([t]), ids=np.asarray([g], dtype=np.int64))
            if cond.guidance_scale != 1.0:
                d2, c2 = apply_cfg(batch, cond)
                eps = handle_cfg(model_forward(model, d2, c2), cond.guidance_scale).epsilon
            else:
                eps = model_forward(model, batch, cond).epsilon
            stats.model_calls += 1
            busy_wait_us(sched_cost_us)
            latent, t = sequential_velocity_step(np.asarray(eps)[0], latent, t, sched, stats.step_stats)
            stats.scheduler_calls += 1
        stats.decodes += 1
        stats.decode_time_us += decode_cost_us
        results.append(GenerationResult(id=g, latent=latent, decoded=decode_stub(latent, decode_cost_us),
                                        iterations_spanned=n))
    return results, stats
