"""CPU oracle of the tiny-VAE (TAESD) decoder (TEST INFRASTRUCTURE ONLY).

The reference has no decoder (decode_stub, src/pipeline.py:86-89, is an identity
copy); the paper decodes retired frames with taesd (madebyollin/taesd, not vendored
in /root/reference).  This restates taesd's published Decoder in torch fp32 with
the same nn.Sequential indices, so ``load_state_dict`` takes taesd_decoder.pth keys:

    Clamp -> conv(4,64) -> ReLU -> Block x3 -> Up2 -> conv(bias=False) -> Block x3
    -> Up2 -> conv -> Block x3 -> Up2 -> conv -> Block -> conv(64,3)
    Block(x) = ReLU(conv(ReLU(conv(ReLU(conv(x))))) + x)     (skip = Identity, 64 -> 64)
    Clamp(x) = tanh(x / 3) * 3

PARITY UNPINNED BY THE REFERENCE (no decoder there, no taesd checkpoint offline):
the device decoder (paper_2511_22009_b200.vae) is compared against this module
within a stated bf16 tolerance (tests/test_gpu_taesd.py).
"""

from __future__ import annotations

import torch
from torch import nn


class Clamp(nn.Module):
    def forward(self, x):
        return torch.tanh(x / 3) * 3


def conv(n_in, n_out, **kw):
    return nn.Conv2d(n_in, n_out, 3, padding=1, **kw)


class Block(nn.Module):
    def __init__(self, n_in, n_out):
        super().__init__()
        self.conv = nn.Sequential(conv(n_in, n_out), nn.ReLU(), conv(n_out, n_out), nn.ReLU(), conv(n_out, n_out))
        self.skip = nn.Identity()
        self.fuse = nn.ReLU()

    def forward(self, x):
        return self.fuse(self.conv(x) + self.skip(x))


def taesd_decoder() -> nn.Sequential:
    return nn.Sequential(
        Clamp(), conv(4, 64), nn.ReLU(),
        Block(64, 64), Block(64, 64), Block(64, 64), nn.Upsample(scale_factor=2), conv(64, 64, bias=False),
        Block(64, 64), Block(64, 64), Block(64, 64), nn.Upsample(scale_factor=2), conv(64, 64, bias=False),
        Block(64, 64), Block(64, 64), Block(64, 64), nn.Upsample(scale_factor=2), conv(64, 64, bias=False),
        Block(64, 64), conv(64, 3),
    )


def decode(state_dict: dict, latents: torch.Tensor) -> torch.Tensor:
    """fp32 CPU decode of [F, 4, 64, 64] latents -> [F, 3, 512, 512]."""
    m = taesd_decoder()
    m.load_state_dict(state_dict)
    with torch.no_grad():
        return m(latents.float().cpu())
