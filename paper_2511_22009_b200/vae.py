"""Tiny-VAE (TAESD) decoder of retired frames on the GPU (csrc/taesd.cu).

The reference decodes nothing: ``decode_stub`` (src/pipeline.py:86-89) copies the
latent and busy-waits ``decode_cost_us``.  The paper pairs the stream batch with
taesd (madebyollin/taesd); this module is that decoder behind the same
``decoded`` slot of ``GenerationResult``: 4x64x64 latents -> 3x512x512 images.

Weights use taesd's ``taesd_decoder.pth`` state-dict names (nn.Sequential
indices), so a real checkpoint loads unchanged; without network access the
tests use ``init_taesd_state`` (seeded, torch-default-style uniform init).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib
from .errors import ParameterError

BLOCKS = (3, 4, 5, 8, 9, 10, 13, 14, 15, 18)  # Sequential indices of the Blocks
UP_CONVS = (7, 12, 17)  # conv(64, 64, bias=False) after each Upsample
LATENT_SHAPE = (4, 64, 64)
IMAGE_SHAPE = (3, 512, 512)


def conv_keys() -> list[tuple[str, str | None]]:
    """(weight key, bias key) of the 33 conv(64, 64) layers in network order."""
    keys = []
    for i in range(3, 19):
        if i in BLOCKS:
            keys += [(f"{i}.conv.{j}.weight", f"{i}.conv.{j}.bias") for j in (0, 2, 4)]
        elif i in UP_CONVS:
            keys.append((f"{i}.weight", None))
    return keys


def init_taesd_state(seed: int = 0) -> dict[str, torch.Tensor]:
    """Seeded random decoder weights in taesd's state-dict layout (fp32, CPU):
    U(-1/sqrt(fan_in), 1/sqrt(fan_in)) like torch's Conv2d default."""
    g = torch.Generator().manual_seed(seed)

    def u(shape, fan_in):
        b = 1.0 / math.sqrt(fan_in)
        return (torch.rand(shape, generator=g, dtype=torch.float64) * 2 - 1).mul_(b).float()

    sd = {"1.weight": u((64, 4, 3, 3), 36), "1.bias": u((64,), 36)}
    for wk, bk in conv_keys():
        sd[wk] = u((64, 64, 3, 3), 576)
        if bk:
            sd[bk] = u((64,), 576)
    sd["19.weight"] = u((3, 64, 3, 3), 576)
    sd["19.bias"] = u((3,), 576)
    return sd


class _Weights(C.Structure):
    _fields_ = [("first_w", C.c_void_p), ("first_b", C.c_void_p), ("conv_w", C.c_void_p * 33),
                ("conv_b", C.c_void_p * 33), ("final_w", C.c_void_p), ("final_b", C.c_void_p)]


_lib.SIGNATURES.update({
    "sf_taesd_act_elems": [C.c_int64, C.c_int32, C.c_int32],
    "sf_conv3x3": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                   C.c_int32, C.c_void_p],
    "sf_taesd_first": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
    "sf_taesd_workspace_bytes": [C.c_int64],
    "sf_taesd_decode": [C.POINTER(_Weights), C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                        C.c_void_p],
})
_lib.RESTYPES.update({"sf_taesd_act_elems": C.c_int64, "sf_taesd_workspace_bytes": C.c_int64})

EPI_NONE, EPI_RELU, EPI_RES_RELU, EPI_RES_RELU_UP2, EPI_FINAL = range(5)


def pack_conv(w: torch.Tensor, n_pad: int | None = None) -> torch.Tensor:
    """torch conv weight [oc][ic][3][3] -> bf16 [9 taps][oc (padded)][ic] (K-major per tap)."""
    oc, ic = w.shape[:2]
    t = w.permute(2, 3, 0, 1).reshape(9, oc, ic)
    if n_pad and n_pad > oc:
        t = torch.cat([t, torch.zeros(9, n_pad - oc, ic, dtype=t.dtype)], 1)
    return t.to(torch.bfloat16).contiguous()


def padded_nhwc(x: torch.Tensor) -> torch.Tensor:
    """[F][64][H][W] -> bf16 [F][H+2][W+2][64] with a zero border (the kernels' layout)."""
    F, Cc, H, W = x.shape
    out = torch.zeros(F, H + 2, W + 2, Cc, dtype=torch.bfloat16, device=x.device)
    out[:, 1:-1, 1:-1] = x.permute(0, 2, 3, 1).to(torch.bfloat16)
    return out


def unpad_nchw(x: torch.Tensor) -> torch.Tensor:
    return x[:, 1:-1, 1:-1].permute(0, 3, 1, 2).float()


def conv3x3(inp: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None, epi: int,
            res: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """One padded-NHWC conv launch (sf_conv3x3); allocates ``out`` (zeroed) if absent."""
    F, Hp, Wp, _ = inp.shape
    H, W = Hp - 2, Wp - 2
    if out is None:
        if epi == EPI_FINAL:
            out = torch.zeros(F, 3, H, W, dtype=torch.float32, device=inp.device)
        elif epi == EPI_RES_RELU_UP2:
            out = torch.zeros(F, 2 * H + 2, 2 * W + 2, 64, dtype=torch.bfloat16, device=inp.device)
        else:
            out = torch.zeros_like(inp)
    _lib.call("sf_conv3x3", inp.data_ptr(), w.data_ptr(), None if bias is None else bias.data_ptr(),
              None if res is None else res.data_ptr(), out.data_ptr(), F, H, W, epi,
              torch.cuda.current_stream().cuda_stream)
    return out


class TinyDecoder:
    """TAESD decoder on the device: ``decode(latents [F,4,64,64] fp32) -> [F,3,512,512]``.

    state_dict  taesd decoder weights (taesd_decoder.pth layout); default: init_taesd_state(seed)
    max_frames  workspace capacity (the padded activations of all four stages, zeroed once)
    """

    def __init__(self, state_dict: dict | None = None, seed: int = 0, max_frames: int = 32, device: str = "cuda",
                 use_graph: bool = True):
        if not torch.cuda.is_available():
            raise RuntimeError("TinyDecoder needs a CUDA device; there is no CPU fallback")
        if max_frames < 1:
            raise ParameterError("max_frames must be >= 1")
        sd = {k: v.detach().float().cpu() for k, v in (state_dict or init_taesd_state(seed)).items()}
        missing = [k for k in self.state_keys() if k not in sd]
        if missing:
            raise ParameterError(f"taesd state dict is missing {missing[:3]}")
        dev = torch.device(device)
        self.device, self.max_frames = dev, int(max_frames)
        self.first_w = sd["1.weight"].contiguous().to(dev)
        self.first_b = sd["1.bias"].contiguous().to(dev)
        self.conv_w, self.conv_b = [], []
        for wk, bk in conv_keys():
            self.conv_w.append(pack_conv(sd[wk]).to(dev))
            self.conv_b.append(None if bk is None else sd[bk].contiguous().to(dev))
        self.final_w = pack_conv(sd["19.weight"], 16).to(dev)
        self.final_b = torch.cat([sd["19.bias"], torch.zeros(13)]).contiguous().to(dev)
        self._w = _Weights()
        self._w.first_w, self._w.first_b = self.first_w.data_ptr(), self.first_b.data_ptr()
        for i, (w, b) in enumerate(zip(self.conv_w, self.conv_b)):
            self._w.conv_w[i] = w.data_ptr()
            self._w.conv_b[i] = None if b is None else b.data_ptr()
        self._w.final_w, self._w.final_b = self.final_w.data_ptr(), self.final_b.data_ptr()
        nbytes = int(_lib.fn("sf_taesd_workspace_bytes")(self.max_frames))
        self.workspace = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        # the 35-launch decode replays as one CUDA graph per (latent, image, F) binding
        self.use_graph = bool(use_graph)
        self._graphs: dict = {}

    @staticmethod
    def state_keys() -> list[str]:
        keys = ["1.weight", "1.bias", "19.weight", "19.bias"]
        for wk, bk in conv_keys():
            keys += [wk] + ([bk] if bk else [])
        return keys

    @staticmethod
    def flops_per_frame() -> float:
        """2*MACs of one 64x64 latent -> 512x512 image decode."""
        f = 2.0 * 64 * 64 * 64 * 4 * 9  # first conv
        for s, n in enumerate((9, 10, 10, 4)):  # conv(64, 64) per stage
            hw = (64 << s) ** 2
            f += n * 2.0 * hw * 64 * 64 * 9
        return f + 2.0 * 512 * 512 * 3 * 64 * 9

    def decode(self, latents: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if latents.dim() == 2:
            latents = latents.view(-1, *LATENT_SHAPE)
        if tuple(latents.shape[1:]) != LATENT_SHAPE:
            raise ParameterError(f"latents must be [F, 4, 64, 64], got {tuple(latents.shape)}")
        F = latents.shape[0]
        if not 1 <= F <= self.max_frames:
            raise ParameterError(f"{F} frames exceed the decoder's max_frames {self.max_frames}")
        lat = latents.to(device=self.device, dtype=torch.float32).contiguous()
        if out is None:
            out = torch.empty(F, *IMAGE_SHAPE, dtype=torch.float32, device=self.device)
        key = (lat.data_ptr(), out.data_ptr(), F)
        g = self._graphs.get(key) if self.use_graph and lat is latents else None
        if g is not None:
            g.replay()
            return out
        self._launch(lat, out, F)
        if self.use_graph and lat is latents and len(self._graphs) < 8 and not torch.cuda.is_current_stream_capturing():
            # capture after one eager run (kernel attributes set); later calls with the same
            # buffers replay it
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch(lat, out, F)
            self._graphs[key] = g
        return out

    def _launch(self, lat: torch.Tensor, out: torch.Tensor, F: int) -> None:
        _lib.call("sf_taesd_decode", C.byref(self._w), lat.data_ptr(), F, self.max_frames,
                  self.workspace.data_ptr(), self.workspace.numel(), out.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)

    __call__ = decode
