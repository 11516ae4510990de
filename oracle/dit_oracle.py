"""CPU oracle of the DiT velocity field (TEST INFRASTRUCTURE ONLY).

The reference (flowpipe) has no network: its VelocityModel plugins are a hash
mock and an affine map (models.py:139-241), so the DiT-S/2 / DiT-XL/2
velocity fields named in BASELINE.json have no reference implementation.
This module restates the standard DiT forward (adaLN-Zero blocks, fixed 2-D
sin-cos positions, tanh-GELU MLP, LayerNorm eps 1e-6 without affine) in plain
torch fp32 on the CPU, behind the reference's VelocityModel contract
(models.py:89-136: row i of eps depends only on row i of the batch).

PARITY UNPINNED BY THE REFERENCE: there are no reference goldens for a DiT.
The device path (paper_2511_22009_b200.dit) is compared against this oracle
within a stated bf16 tolerance (tests/test_gpu_dit_forward.py), and this
oracle's own conventions are pinned by self-recorded properties in
tests/test_dit_oracle.py (shape, row independence, determinism).
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def timestep_features(t: torch.Tensor, dim: int = 256) -> torch.Tensor:
    """sinusoid(1000 t): cos | sin over freqs exp(-ln(1e4) k / half)."""
    half = dim // 2
    freqs = torch.exp(-math.log(10000.0) * torch.arange(half, dtype=torch.float32, device=t.device) / half)
    args = (1000.0 * t.to(torch.float64)).to(torch.float32)[:, None] * freqs[None]
    return torch.cat([torch.cos(args), torch.sin(args)], dim=-1)


def _modulate(x, shift, scale):
    return x * (1 + scale[:, None, :]) + shift[:, None, :]


@torch.no_grad()
def dit_forward(params: dict, x: torch.Tensor, t: torch.Tensor, emb: torch.Tensor, heads: int,
                patch: int = 2, eps: float = 1e-6) -> torch.Tensor:
    """x [B, C, H, W] fp32, t [B] (flow time), emb [B, E] -> eps [B, C, H, W]."""
    B, Cc, Hh, Ww = x.shape
    H = params["patch_b"].numel()
    tok = F.conv2d(x.float(), params["patch_w"], params["patch_b"], stride=patch)  # [B, H, gh, gw]
    gh, gw = tok.shape[-2:]
    h = tok.flatten(2).transpose(1, 2) + params["pos_embed"][None]
    f = timestep_features(t, params["t_w1"].shape[1])
    temb = F.linear(F.silu(F.linear(f, params["t_w1"], params["t_b1"])), params["t_w2"], params["t_b2"])
    c = temb + F.linear(emb.float(), params["y_w"], params["y_b"])
    sc = F.silu(c)
    d = H // heads
    for blk in params["blocks"]:
        sh_msa, sc_msa, g_msa, sh_mlp, sc_mlp, g_mlp = F.linear(sc, blk["ada_w"], blk["ada_b"]).chunk(6, dim=1)
        a = _modulate(F.layer_norm(h, (H,), eps=eps), sh_msa, sc_msa)
        qkv = F.linear(a, blk["qkv_w"], blk["qkv_b"]).reshape(B, -1, 3, heads, d).permute(2, 0, 3, 1, 4)
        o = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2])
        o = o.transpose(1, 2).reshape(B, -1, H)
        h = h + g_msa[:, None, :] * F.linear(o, blk["proj_w"], blk["proj_b"])
        m = _modulate(F.layer_norm(h, (H,), eps=eps), sh_mlp, sc_mlp)
        m = F.linear(F.gelu(F.linear(m, blk["fc1_w"], blk["fc1_b"]), approximate="tanh"),
                     blk["fc2_w"], blk["fc2_b"])
        h = h + g_mlp[:, None, :] * m
    shift, scale = F.linear(sc, params["final_ada_w"], params["final_ada_b"]).chunk(2, dim=1)
    h = _modulate(F.layer_norm(h, (H,), eps=eps), shift, scale)
    out = F.linear(h, params["final_w"], params["final_b"])  # [B, T, p*p*C]
    out = out.reshape(B, gh, gw, patch, patch, Cc)
    return torch.einsum("nhwpqc->nchpwq", out).reshape(B, Cc, gh * patch, gw * patch)


def params_to(params: dict, device) -> dict:
    """The same parameters on another device (e.g. to run this fp32 reference on a
    GPU for the DiT-XL/2-sized parity test, where the CPU is too slow)."""
    out = {k: (v.to(device) if torch.is_tensor(v) else v) for k, v in params.items() if k != "blocks"}
    out["blocks"] = [{k: v.to(device) for k, v in b.items()} for b in params["blocks"]]
    return out
