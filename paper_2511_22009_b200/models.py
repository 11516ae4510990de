"""Velocity-model plugin boundary (drop-in for flowpipe models.py).

* ``VelocityModel``: the reference ABC (models.py:89-136) -- ``forward``
  validates, burns the declared cost, then calls ``_compute``; row i of the
  output depends only on row i of the input.
* ``SeededMockModel``: the reference's hash mock (models.py:199-241) computed
  on the GPU (device blake2b row keys + splitmix64 expansion, kernel K12),
  bit-exact with the reference.
* ``DiTVelocityModel``: the DiT-S/2 (or XL/2) velocity field of BASELINE.json
  on the native runtime (dit.py).
* ``apply_cfg`` / ``handle_cfg``: classifier-free guidance doubling and
  combine (models.py:244-296); the combine runs on the GPU.
"""

from __future__ import annotations

import time
from abc import ABC, abstractmethod
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ParameterError, StateError
from .velocity import LatentBatch, _is_torch, _to_device


@dataclass(frozen=True)
class Conditioning:
    """models.py:33-55."""

    embedding: np.ndarray
    guidance_scale: float = 1.0
    negative_embedding: np.ndarray | None = None
    row_embeddings: np.ndarray | None = None

    @property
    def embed_dim(self) -> int:
        return len(self.embedding)

    def embedding_for_row(self, row: int) -> np.ndarray:
        if self.row_embeddings is not None:
            return self.row_embeddings[row]
        return self.embedding


def make_conditioning(embedding, guidance_scale: float = 1.0, negative_embedding=None) -> Conditioning:
    """models.py:58-73."""
    if guidance_scale < 0.0:
        raise ParameterError(f"guidance_scale must be >= 0, got {guidance_scale}")
    emb = np.asarray(embedding, dtype=np.float64)
    neg = None if negative_embedding is None else np.asarray(negative_embedding, dtype=np.float64)
    if neg is not None and neg.shape != emb.shape:
        raise ParameterError(f"negative embedding length {neg.shape} != embedding length {emb.shape}")
    return Conditioning(embedding=emb, guidance_scale=guidance_scale, negative_embedding=neg)


@dataclass(frozen=True)
class ModelOutput:
    """models.py:76-86."""

    epsilon: object
    aux: list | None = None


def busy_wait_us(us: float) -> None:
    """Declared-cost injection of the reference models (timing.py:15-24)."""
    if us <= 0.0:
        return
    end = time.perf_counter() + us * 1e-6
    while time.perf_counter() < end:
        pass


class VelocityModel(ABC):
    """(latents, timesteps, conditioning) -> noise prediction (models.py:89-136)."""

    dim: int
    embed_dim: int
    cost_us: float

    def __init__(self, dim: int, embed_dim: int, cost_us: float = 0.0):
        if dim < 1 or embed_dim < 1:
            raise ParameterError("dim and embed_dim must be >= 1")
        if cost_us < 0.0:
            raise ParameterError(f"cost_us must be >= 0, got {cost_us}")
        self.dim, self.embed_dim, self.cost_us = dim, embed_dim, cost_us

    def forward(self, batch: LatentBatch, cond: Conditioning) -> ModelOutput:
        self._check(batch, cond)
        busy_wait_us(self.cost_us)
        return self._compute(batch, cond)

    def _check(self, batch: LatentBatch, cond: Conditioning) -> None:
        if batch.batch_size == 0:
            raise ParameterError("batch must be non-empty")
        if batch.dim != self.dim:
            raise ParameterError(f"latent dim {batch.dim} != model dim {self.dim}")
        if cond.embed_dim != self.embed_dim:
            raise ParameterError(f"embedding length {cond.embed_dim} != model embed_dim {self.embed_dim}")
        if cond.row_embeddings is not None and len(cond.row_embeddings) != batch.batch_size:
            raise ParameterError(f"{len(cond.row_embeddings)} row embeddings for batch of {batch.batch_size}")

    @abstractmethod
    def _compute(self, batch: LatentBatch, cond: Conditioning) -> ModelOutput:
        """Pure computation (no cost injection)."""


def _row_embs(batch: LatentBatch, cond: Conditioning) -> np.ndarray:
    if cond.row_embeddings is not None:
        return np.asarray(cond.row_embeddings, dtype=np.float64)
    return np.tile(np.asarray(cond.embedding, dtype=np.float64), (batch.batch_size, 1))


def _host_if(like, t: torch.Tensor):
    return t if _is_torch(like) else t.cpu().numpy()


class SeededMockModel(VelocityModel):
    """Hash-derived outputs in [-1, 1) (models.py:199-241), computed on the GPU:
    kernel K12 = blake2b-64 row key of (seed, id, round(t*1e9), embedding) +
    splitmix64 expansion.  Latent values are ignored, like the reference."""

    def __init__(self, dim: int = 16, embed_dim: int = 8, cost_us: float = 0.0, seed: int = 0,
                 aux_scales: tuple = ()):
        super().__init__(dim=dim, embed_dim=embed_dim, cost_us=cost_us)
        self.seed = int(seed)
        self.aux_scales = aux_scales

    def eps_device(self, ids: torch.Tensor, ts: torch.Tensor, row_embs: torch.Tensor) -> torch.Tensor:
        B = ids.numel()
        st = torch.cuda.current_stream().cuda_stream
        keys = torch.empty(B, dtype=torch.int64, device=ids.device)
        _lib.call("sf_mock_keys", self.seed, ids.data_ptr(), ts.data_ptr(), row_embs.data_ptr(), B,
                  self.embed_dim, keys.data_ptr(), st)
        out = torch.empty(B, self.dim, dtype=torch.float64, device=ids.device)
        _lib.call("sf_mock_eps", keys.data_ptr(), B, self.dim, out.data_ptr(), st)
        return out

    def _compute(self, batch: LatentBatch, cond: Conditioning) -> ModelOutput:
        ids = _to_device(batch.ids, torch.int64)
        ts = _to_device(batch.timesteps, torch.float64)
        embs = _to_device(_row_embs(batch, cond), torch.float64)
        eps = self.eps_device(ids, ts, embs)
        aux = [scale * eps for scale in self.aux_scales] if self.aux_scales else None
        eps_o = _host_if(batch.data, eps)
        return ModelOutput(epsilon=eps_o, aux=None if aux is None else [_host_if(batch.data, a) for a in aux])


class AnalyticLinearModel(VelocityModel):
    """Closed-form model eps_i = A x_i + t_i b (models.py:139-185) on the GPU (kernel
    K13): fp64, one output element per thread as a sequential dot product, so a row's
    result does not depend on the batch it arrives in (models.py:142-146).  Defaults
    A = 0.1 I, b = 0.05 (models.py:162-165); conditioning does not enter the map."""

    def __init__(self, dim: int = 16, embed_dim: int = 8, cost_us: float = 0.0, a_matrix=None, b_vector=None,
                 aux_scales: tuple = ()):
        super().__init__(dim=dim, embed_dim=embed_dim, cost_us=cost_us)
        a_matrix = 0.1 * np.eye(dim) if a_matrix is None else a_matrix
        b_vector = 0.05 * np.ones(dim) if b_vector is None else b_vector
        self.a_matrix = np.asarray(a_matrix, dtype=np.float64)
        self.b_vector = np.asarray(b_vector, dtype=np.float64)
        if self.a_matrix.shape != (dim, dim):
            raise ParameterError(f"a_matrix shape {self.a_matrix.shape} != ({dim}, {dim})")
        if self.b_vector.shape != (dim,):
            raise ParameterError(f"b_vector shape {self.b_vector.shape} != ({dim},)")
        self.aux_scales = aux_scales
        self._a_dev = None

    def _device_ab(self):
        if self._a_dev is None:
            self._a_dev = (torch.from_numpy(self.a_matrix).cuda(), torch.from_numpy(self.b_vector).cuda())
        return self._a_dev

    def _compute(self, batch: LatentBatch, cond: Conditioning) -> ModelOutput:
        a_dev, b_dev = self._device_ab()
        if _is_torch(batch.data):
            xdt = torch.float32 if batch.data.dtype == torch.float32 else torch.float64
        else:
            xdt = torch.float32 if np.asarray(batch.data).dtype == np.float32 else torch.float64
        x = _to_device(batch.data, xdt).contiguous()
        ts = _to_device(batch.timesteps, torch.float64)
        B = x.shape[0]
        out = torch.empty(B, self.dim, dtype=torch.float64, device=x.device)
        _lib.call("sf_analytic_eps", a_dev.data_ptr(), b_dev.data_ptr(), x.data_ptr(),
                  _lib.SF_F32 if xdt == torch.float32 else _lib.SF_F64, ts.data_ptr(), B, self.dim, out.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        aux = [scale * out for scale in self.aux_scales] if self.aux_scales else None
        return ModelOutput(epsilon=_host_if(batch.data, out),
                           aux=None if aux is None else [_host_if(batch.data, a) for a in aux])


class DiTVelocityModel(VelocityModel):
    """DiT velocity field (dit.py) as a VelocityModel plugin.  ``forward`` runs
    the native sf_dit_forward; StreamBatch uses the fused sf_dit_stream_step."""

    def __init__(self, cfg=None, seed: int = 0, max_rows: int = 8, params: dict | None = None,
                 bias_std: float = 0.0, cost_us: float = 0.0):
        from .dit import DIT_S2, DeviceDiT, init_dit_params

        cfg = cfg or DIT_S2
        super().__init__(dim=cfg.dim, embed_dim=cfg.embed_dim, cost_us=cost_us)
        self.cfg = cfg
        self.params = params if params is not None else init_dit_params(cfg, seed=seed, bias_std=bias_std)
        self.device_model = DeviceDiT(self.params, cfg, max_rows=max_rows)

    @property
    def max_rows(self) -> int:
        return self.device_model.max_rows

    def _compute(self, batch: LatentBatch, cond: Conditioning) -> ModelOutput:
        x = _to_device(batch.data, torch.float32)
        ts = _to_device(batch.timesteps, torch.float64)
        embs = _to_device(_row_embs(batch, cond), torch.float64)
        outs = []
        for r0 in range(0, x.shape[0], self.max_rows):
            r1 = min(r0 + self.max_rows, x.shape[0])
            outs.append(self.device_model.forward(x[r0:r1], ts[r0:r1], embs[r0:r1]))
        eps = torch.cat(outs) if len(outs) > 1 else outs[0]
        return ModelOutput(epsilon=_host_if(batch.data, eps))


def apply_cfg(batch: LatentBatch, cond: Conditioning):
    """[uncond; cond] doubling (models.py:244-275); identity when w == 1."""
    w = cond.guidance_scale
    if w == 1.0:
        return batch, cond
    b = batch.batch_size
    neg = cond.negative_embedding if cond.negative_embedding is not None else np.zeros_like(cond.embedding)
    row_emb = np.concatenate([np.tile(neg, (b, 1)), np.tile(cond.embedding, (b, 1))], axis=0)
    cat = torch.cat if _is_torch(batch.data) else np.concatenate
    doubled = LatentBatch(data=cat([batch.data, batch.data]), timesteps=cat([batch.timesteps, batch.timesteps]),
                          ids=cat([batch.ids, batch.ids]))
    paired = Conditioning(embedding=cond.embedding, guidance_scale=w, negative_embedding=cond.negative_embedding,
                          row_embeddings=row_emb)
    return doubled, paired


def _combine(mat, w: float):
    rows = mat.shape[0]
    half = rows // 2
    t = _to_device(mat)
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    out = torch.empty(half, t.shape[1], dtype=t.dtype, device=t.device)
    _lib.call("sf_cfg_combine", t.data_ptr(), _lib.SF_F64 if t.dtype == torch.float64 else _lib.SF_F32,
              half, t.shape[1], float(w), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return _host_if(mat, out)


def handle_cfg(out: ModelOutput, w: float) -> ModelOutput:
    """eps_u + w (eps_c - eps_u) per sample on the GPU (models.py:278-296)."""
    rows = out.epsilon.shape[0]
    if rows % 2 != 0:
        raise StateError(f"guided output has odd row count {rows}; halves cannot pair")
    aux = None if out.aux is None else [_combine(a, w) for a in out.aux]
    return ModelOutput(epsilon=_combine(out.epsilon, w), aux=aux)
