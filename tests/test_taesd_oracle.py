"""CPU checks of the TAESD decoder's weight layout and oracle (no GPU)."""

import torch

from oracle.taesd_oracle import decode, taesd_decoder
from paper_2511_22009_b200.vae import TinyDecoder, conv_keys, init_taesd_state, pack_conv


def test_state_dict_layout_is_taesd():
    """init_taesd_state / TinyDecoder use taesd_decoder.pth's nn.Sequential keys."""
    keys = set(taesd_decoder().state_dict().keys())
    assert keys == set(init_taesd_state(0).keys()) == set(TinyDecoder.state_keys())
    assert len(conv_keys()) == 33 and sum(b is None for _, b in conv_keys()) == 3


def test_pack_conv_tap_major():
    w = torch.arange(3 * 64 * 9, dtype=torch.float32).view(3, 64, 3, 3)
    p = pack_conv(w, 16).float()
    assert p.shape == (9, 16, 64)
    assert p[4, 2, 5] == w[2, 5, 1, 1].to(torch.bfloat16).float() and p[:, 3:].abs().max() == 0


def test_oracle_shapes_and_determinism():
    sd = init_taesd_state(2)
    lat = torch.randn(1, 4, 64, 64, generator=torch.Generator().manual_seed(0))
    a = decode(sd, lat)
    assert a.shape == (1, 3, 512, 512) and torch.isfinite(a).all()
    assert torch.equal(a, decode(init_taesd_state(2), lat))


def test_flops_per_frame():
    assert abs(TinyDecoder.flops_per_frame() / 1e9 - 141.35) < 0.01
