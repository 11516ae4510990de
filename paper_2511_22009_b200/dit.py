"""DiT velocity field behind the reference's ``VelocityModel`` plugin boundary.

The reference ships no network (its models are a hash mock and an affine map,
flowpipe models.py:139-241); BASELINE.json names a random-init DiT-S/2 (and
DiT-XL/2) over a 64x64x4 latent.  Conventions (fixed here once):

* latent flat index = c*4096 + h*64 + w  (x viewed as [B, 4, 64, 64]);
* model time = 1000 * t (flow time t in [0, 1]);
* conditioning = the reference's E=8 embedding vector (models.py:33-55) through
  Linear(E -> hidden) (replaces DiT's class-label table);
* every Linear / Conv weight ~ N(0, 0.02^2) (adaLN and final layer included,
  so eps is not identically zero), biases 0 unless ``bias_std`` > 0; all
  weights are rounded to bf16 once, so the device path and the CPU oracle
  (oracle/dit_oracle.py) use identical parameter values;
* output = 4 channels (eps only), unpatchify feature f = (p*2 + q)*4 + c.

Compute runs only through ``libstreamflow.so`` (sf_dit_* C ABI); there is no
CPU path here.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass(frozen=True)
class DiTConfig:
    depth: int = 12
    hidden: int = 384
    heads: int = 6
    patch: int = 2
    in_ch: int = 4
    latent_hw: int = 64
    embed_dim: int = 8
    freq_dim: int = 256
    mlp_ratio: int = 4
    ln_eps: float = 1e-6

    @property
    def mlp_hidden(self) -> int:
        return self.hidden * self.mlp_ratio

    @property
    def tokens(self) -> int:
        return (self.latent_hw // self.patch) ** 2

    @property
    def dim(self) -> int:
        return self.in_ch * self.latent_hw * self.latent_hw

    @property
    def out_features(self) -> int:
        return self.patch * self.patch * self.in_ch

    def flops_per_row(self) -> float:
        """Algorithmic FLOPs of one velocity evaluation of one latent (2*M*N*K per
        GEMM, 4*T^2*d per attention layer, embeddings included)."""
        T, H, Fm = self.tokens, self.hidden, self.mlp_hidden
        per_block = 2 * T * H * (3 * H + H + Fm + Fm) + 4 * T * T * H
        ada = 2 * H * (6 * H * self.depth + 2 * H)
        emb = 2 * (self.freq_dim * H + H * H + self.embed_dim * H)
        io = 2 * T * H * (self.patch ** 2 * self.in_ch) * 2
        return float(self.depth * per_block + ada + emb + io)


DIT_S2 = DiTConfig()
DIT_XL2 = DiTConfig(depth=28, hidden=1152, heads=16)


def _sincos_1d(dim: int, pos: np.ndarray) -> np.ndarray:
    omega = 1.0 / 10000 ** (np.arange(dim // 2, dtype=np.float64) / (dim / 2.0))
    out = np.einsum("m,d->md", pos.reshape(-1), omega)
    return np.concatenate([np.sin(out), np.cos(out)], axis=1)


def pos_embed_2d(dim: int, grid: int) -> np.ndarray:
    """Fixed 2-D sin-cos position table [grid*grid, dim] (DiT / MAE convention:
    first half encodes the row index, second half the column index)."""
    gh, gw = np.meshgrid(np.arange(grid, dtype=np.float64), np.arange(grid, dtype=np.float64), indexing="ij")
    return np.concatenate([_sincos_1d(dim // 2, gh), _sincos_1d(dim // 2, gw)], axis=1).astype(np.float32)


def init_dit_params(cfg: DiTConfig = DIT_S2, seed: int = 0, std: float = 0.02,
                    bias_std: float = 0.0) -> dict:
    """Canonical fp32 CPU parameters (bf16-representable weights)."""
    g = torch.Generator().manual_seed(seed)
    H, E, F, P, Cc = cfg.hidden, cfg.embed_dim, cfg.freq_dim, cfg.patch, cfg.in_ch

    def w(*shape):
        return (torch.randn(*shape, generator=g) * std).to(torch.bfloat16).float()

    def b(n):
        if bias_std == 0.0:
            return torch.zeros(n)
        return torch.randn(n, generator=g) * bias_std

    p = {
        "patch_w": w(H, Cc, P, P), "patch_b": b(H),
        "pos_embed": torch.from_numpy(pos_embed_2d(H, cfg.latent_hw // P)),
        "t_w1": w(H, F), "t_b1": b(H), "t_w2": w(H, H), "t_b2": b(H),
        "y_w": w(H, E), "y_b": b(H),
        "final_ada_w": w(2 * H, H), "final_ada_b": b(2 * H),
        "final_w": w(P * P * Cc, H), "final_b": b(P * P * Cc),
        "blocks": [],
    }
    for _ in range(cfg.depth):
        p["blocks"].append({
            "ada_w": w(6 * H, H), "ada_b": b(6 * H),
            "qkv_w": w(3 * H, H), "qkv_b": b(3 * H),
            "proj_w": w(H, H), "proj_b": b(H),
            "fc1_w": w(cfg.mlp_hidden, H), "fc1_b": b(cfg.mlp_hidden),
            "fc2_w": w(H, cfg.mlp_hidden), "fc2_b": b(H),
        })
    return p


class _Cfg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("depth", "hidden", "heads", "patch", "in_ch", "latent_hw",
                                          "embed_dim", "freq_dim", "mlp_hidden")] + [("ln_eps", C.c_float)]


class _Weights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "patch_w", "patch_b", "pos_embed", "t_w1t", "t_b1", "t_w2t", "t_b2", "y_wt", "y_b", "ada_w", "ada_b",
        "qkv_w", "qkv_b", "proj_w", "proj_b", "fc1_w", "fc1_b", "fc2_w", "fc2_b", "final_w", "final_b")]


_lib.SIGNATURES.update({
    "sf_dit_workspace_bytes": [C.POINTER(_Cfg), C.c_int64],
    "sf_dit_mod_stride": [C.POINTER(_Cfg)],
    "sf_dit_create": [C.POINTER(_Cfg), C.POINTER(_Weights), C.c_int64, C.c_void_p, C.c_int64,
                      C.POINTER(C.c_void_p)],
    "sf_dit_destroy": [C.c_void_p],
    "sf_dit_forward": [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    "sf_dit_stream_step": [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p,
                           C.c_uint64, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p],
    "sf_dit_stream_reset": [C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                            C.c_uint64, C.c_void_p],
    "sf_dit_profile_step": [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p,
                            C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    "sf_dit_launch_count": [C.c_void_p],
    "sf_dit_graph_release": [C.c_void_p, C.c_void_p],
    "sf_dit_graph_count": [C.c_void_p],
})
_lib.RESTYPES["sf_dit_launch_count"] = C.c_int64
_lib.RESTYPES["sf_dit_graph_count"] = C.c_int64

PROFILE_CLASSES = ("prepare", "cond", "adaln_gemm", "patch_embed_ln", "qkv_gemm", "attention",
                   "proj_gemm_res_ln", "fc1_gemm_gelu", "fc2_gemm_res_ln", "final_euler_refill", "block_tail")


class DeviceDiT:
    """bf16 weights resident in HBM + the native runtime handle (sf_dit)."""

    def __init__(self, params: dict, cfg: DiTConfig = DIT_S2, max_rows: int = 8, device: str = "cuda"):
        if not torch.cuda.is_available():
            raise RuntimeError("DeviceDiT needs a CUDA device (sm_100a); there is no CPU fallback")
        _lib.load()
        self.cfg, self.max_rows, self.device = cfg, int(max_rows), device
        bf, f32 = torch.bfloat16, torch.float32

        def d(t, dt):
            return t.to(device=device, dtype=dt).contiguous()

        blocks = params["blocks"]
        self._t = {
            "patch_w": d(params["patch_w"].reshape(cfg.hidden, -1), bf),
            "patch_b": d(params["patch_b"], f32),
            "pos_embed": d(params["pos_embed"], f32),
            "t_w1t": d(params["t_w1"].t(), bf), "t_b1": d(params["t_b1"], f32),
            "t_w2t": d(params["t_w2"].t(), bf), "t_b2": d(params["t_b2"], f32),
            "y_wt": d(params["y_w"].t(), bf), "y_b": d(params["y_b"], f32),
            "ada_w": d(torch.cat([b_["ada_w"] for b_ in blocks] + [params["final_ada_w"]]), bf),
            "ada_b": d(torch.cat([b_["ada_b"] for b_ in blocks] + [params["final_ada_b"]]), f32),
            "final_w": d(params["final_w"], bf), "final_b": d(params["final_b"], f32),
        }
        for name in ("qkv", "proj", "fc1", "fc2"):
            self._t[name + "_w"] = d(torch.stack([b_[name + "_w"] for b_ in blocks]), bf)
            self._t[name + "_b"] = d(torch.stack([b_[name + "_b"] for b_ in blocks]), f32)
        self._cfg = _Cfg(cfg.depth, cfg.hidden, cfg.heads, cfg.patch, cfg.in_ch, cfg.latent_hw,
                         cfg.embed_dim, cfg.freq_dim, cfg.mlp_hidden, cfg.ln_eps)
        self._w = _Weights(*[self._t[n].data_ptr() for n, _ in _Weights._fields_])
        ws = int(_lib.fn("sf_dit_workspace_bytes")(C.byref(self._cfg), self.max_rows))
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=device)
        self._h = C.c_void_p()
        _lib.call("sf_dit_create", C.byref(self._cfg), C.byref(self._w), self.max_rows,
                  self.workspace.data_ptr(), ws, C.byref(self._h))
        self.weight_bytes = sum(t.numel() * t.element_size() for t in self._t.values())

    @property
    def handle(self):
        return self._h

    def forward(self, x: torch.Tensor, ts: torch.Tensor, row_embs: torch.Tensor, out: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
        """eps = DiT(x, 1000 t, emb) for ``rows`` latents.  x: [rows, D] (or
        [rows, C, H, W]) fp32 CUDA; ts: [rows] fp64; row_embs: [rows, E] fp64."""
        rows = x.shape[0]
        if rows > self.max_rows:
            raise ValueError(f"{rows} rows > max_rows {self.max_rows}")
        x = x.reshape(rows, -1).to(torch.float32).contiguous()
        ts = ts.to(device=x.device, dtype=torch.float64).contiguous()
        row_embs = row_embs.to(device=x.device, dtype=torch.float64).contiguous()
        if out is None:
            out = torch.empty(rows, self.cfg.dim, dtype=torch.float32, device=x.device)
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _lib.call("sf_dit_forward", self._h, rows, x.data_ptr(), ts.data_ptr(), row_embs.data_ptr(),
                  out.data_ptr(), st)
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        hv = getattr(h, "value", None)
        if hv:
            # null the handle object in place first: holders of it (a StreamBatch in the same
            # garbage cycle, finalized after this model) then see NULL, never a freed handle
            h.value = None
            try:
                _lib.fn("sf_dit_destroy")(hv)
            except Exception:
                pass
