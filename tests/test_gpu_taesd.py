"""Tiny-VAE (TAESD) decoder on sm_100a (csrc/taesd.cu) vs torch fp32.

Per-layer: the padded-NHWC tcgen05 conv against F.conv2d on the same bf16-rounded
inputs/weights (fp32 accumulate; output rounded to bf16 once) for every epilogue.
Whole decoder: against oracle/taesd_oracle.py (fp32 CPU, taesd's nn.Sequential);
bf16 activations through 34 convs -> normalised bound max 3e-2 / mean 5e-3 of max|img|.
"""

import pytest
import torch
import torch.nn.functional as Fn

from paper_2511_22009_b200 import vae as V

pytestmark = pytest.mark.gpu


def _rb(t):
    return t.to(torch.bfloat16).float()


def _ref(x, w, b, epi, res=None):
    torch.backends.cudnn.allow_tf32 = False
    y = Fn.conv2d(x.double(), w.double(), None if b is None else b.double(), padding=1)
    if res is not None:
        y = y + res.double()
    if epi != V.EPI_NONE and epi != V.EPI_FINAL:
        y = y.clamp_min(0)
    if epi == V.EPI_RES_RELU_UP2:
        y = y.repeat_interleave(2, 2).repeat_interleave(2, 3)
    return y.float()


def _check(got, want, tol_max=1e-2, tol_mean=1e-3):
    scale = want.abs().max().item()
    err = (got - want).abs()
    assert err.max().item() <= tol_max * scale, (err.max().item(), scale)
    assert err.mean().item() <= tol_mean * scale, (err.mean().item(), scale)


@pytest.mark.parametrize("F,H,W", [(2, 64, 64), (1, 128, 128), (3, 16, 200)])
@pytest.mark.parametrize("epi", [V.EPI_NONE, V.EPI_RELU, V.EPI_RES_RELU, V.EPI_RES_RELU_UP2])
def test_conv_epilogues(F, H, W, epi):
    g = torch.Generator(device="cuda").manual_seed(F * 1000 + H + epi)
    x = _rb(torch.randn(F, 64, H, W, device="cuda", generator=g))
    w = _rb(torch.randn(64, 64, 3, 3, device="cuda", generator=g) / 24)
    b = torch.randn(64, device="cuda", generator=g) * 0.1
    res = _rb(torch.randn(F, 64, H, W, device="cuda", generator=g)) if epi >= V.EPI_RES_RELU else None
    xin = V.padded_nhwc(x)
    rin = V.padded_nhwc(res) if res is not None else None
    out = V.conv3x3(xin, V.pack_conv(w.cpu()).cuda(), None if epi == V.EPI_NONE else b, epi, rin)
    got = V.unpad_nchw(out)
    want = _ref(x, w, None if epi == V.EPI_NONE else b, epi, res)
    _check(got, want)
    # borders stay zero (the next layer's padding)
    assert out[:, 0].abs().max() == 0 and out[:, -1].abs().max() == 0
    assert out[:, :, 0].abs().max() == 0 and out[:, :, -1].abs().max() == 0


def test_conv_final_three_channels():
    g = torch.Generator(device="cuda").manual_seed(7)
    x = _rb(torch.randn(2, 64, 96, 160, device="cuda", generator=g))
    w = _rb(torch.randn(3, 64, 3, 3, device="cuda", generator=g) / 24)
    b = torch.randn(3, device="cuda", generator=g)
    bp = torch.cat([b, torch.zeros(13, device="cuda")])
    got = V.conv3x3(V.padded_nhwc(x), V.pack_conv(w.cpu(), 16).cuda(), bp, V.EPI_FINAL)
    _check(got, _ref(x, w, b, V.EPI_FINAL), tol_max=1e-4, tol_mean=1e-5)  # fp32 output: accumulate-order only


def test_first_conv_clamp():
    g = torch.Generator(device="cuda").manual_seed(3)
    lat = torch.randn(3, 4, 64, 64, device="cuda", generator=g) * 4
    w = torch.randn(64, 4, 3, 3, device="cuda", generator=g) / 6
    b = torch.randn(64, device="cuda", generator=g) * 0.1
    out = torch.zeros(3, 66, 66, 64, dtype=torch.bfloat16, device="cuda")
    from paper_2511_22009_b200 import _lib
    _lib.call("sf_taesd_first", lat.data_ptr(), w.data_ptr(), b.data_ptr(), out.data_ptr(), 3,
              torch.cuda.current_stream().cuda_stream)
    want = Fn.conv2d(torch.tanh(lat.double() / 3) * 3, w.double(), b.double(), padding=1).clamp_min(0).float()
    _check(V.unpad_nchw(out), want)


@pytest.mark.parametrize("F", [1, 3])
def test_decoder_matches_oracle(F):
    from oracle.taesd_oracle import decode

    sd = V.init_taesd_state(5)
    dec = V.TinyDecoder(sd, max_frames=4)
    g = torch.Generator().manual_seed(F)
    lat = torch.randn(F, 4, 64, 64, generator=g)
    got = dec.decode(lat.cuda()).cpu()
    want = decode(sd, lat)
    assert got.shape == (F, 3, 512, 512)
    _check(got, want, tol_max=3e-2, tol_mean=5e-3)


def test_decoder_frame_independence_and_reuse():
    """Frame f's image depends only on latent f, for any F <= max_frames and across calls."""
    dec = V.TinyDecoder(seed=1, max_frames=4)
    g = torch.Generator(device="cuda").manual_seed(9)
    lat = torch.randn(4, 4, 64, 64, device="cuda", generator=g)
    full = dec.decode(lat).clone()
    one = dec.decode(lat[2:3]).clone()
    assert torch.equal(full[2:3], one)
    again = dec.decode(lat)
    assert torch.equal(full, again)


def test_stream_batch_decodes_retired_frames():
    """StreamBatch(decoder=...) returns each retired frame's image = decode(latent)."""
    import numpy as np

    import paper_2511_22009_b200 as sf

    sched = sf.build_time_window_schedule(inference_steps=2)
    model = sf.SeededMockModel(dim=16384, seed=4)
    cond = sf.make_conditioning(np.zeros(8))
    dec = V.TinyDecoder(seed=2, max_frames=2)
    sb = sf.StreamBatch(model, sched, 2, num_streams=2, cond=cond, seed=[1, 2], m=2, dtype=np.float32, decoder=dec)
    got = []
    while not sb.done():
        got += sb.step()
    assert [r.id for _, r in got] == [0, 0, 1, 1]
    for _, r in got:
        want = dec.decode(torch.from_numpy(r.latent).cuda().view(1, 4, 64, 64)).cpu().numpy()[0]
        assert r.decoded.image.shape == (3, 512, 512)
        assert np.array_equal(r.decoded.image, want)
