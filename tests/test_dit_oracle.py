"""Self-pins of the DiT CPU oracle (there are no reference goldens for a DiT:
the reference package has no network).  Checks the
VelocityModel contract and the conventions fixed in dit.py: shapes, row
independence (models.py:92-96), determinism, the 2-D sin-cos table, the
unpatchify channel order and the FLOP count used for the roofline."""

import math

import numpy as np
import torch

from oracle.dit_oracle import dit_forward, timestep_features
from paper_2511_22009_b200.dit import DIT_S2, DIT_XL2, DiTConfig, init_dit_params, pos_embed_2d

TINY = DiTConfig(depth=2, hidden=128, heads=2, latent_hw=16)


def test_forward_shape_determinism_row_independence():
    p = init_dit_params(TINY, seed=1, bias_std=0.02)
    g = torch.Generator().manual_seed(0)
    x = torch.randn(3, 4, 16, 16, generator=g)
    t = torch.tensor([0.0, 0.25, 0.75], dtype=torch.float64)
    e = torch.randn(3, 8, generator=g, dtype=torch.float64)
    a = dit_forward(p, x, t, e, heads=2)
    assert a.shape == (3, 4, 16, 16)
    assert torch.equal(a, dit_forward(p, x, t, e, heads=2))
    one = dit_forward(p, x[1:2], t[1:2], e[1:2], heads=2)
    assert torch.allclose(one, a[1:2], atol=1e-5, rtol=1e-5)
    assert a.abs().max() > 0  # random-init adaLN / final layer: eps is not identically zero


def test_weights_are_bf16_representable_and_seeded():
    p1 = init_dit_params(TINY, seed=7)
    p2 = init_dit_params(TINY, seed=7)
    for k in ("patch_w", "t_w1", "final_w"):
        assert torch.equal(p1[k], p2[k])
        assert torch.equal(p1[k], p1[k].to(torch.bfloat16).float())
    assert torch.equal(p1["blocks"][0]["qkv_b"], torch.zeros(3 * TINY.hidden))


def test_pos_embed_and_timestep_features():
    pe = pos_embed_2d(8, 4)
    assert pe.shape == (16, 8)
    # token (i, j): first half encodes the row i, second half the column j
    # each half is [sin(pos*w_k) | cos(pos*w_k)]
    assert np.allclose(pe[1 * 4 + 0, 4:6], [0.0, 0.0]) and np.allclose(pe[1 * 4 + 0, 6:8], [1.0, 1.0])
    assert np.allclose(pe[0 * 4 + 1, 0:2], [0.0, 0.0]) and np.allclose(pe[0 * 4 + 1, 2:4], [1.0, 1.0])
    assert abs(pe[1 * 4 + 0, 0] - math.sin(1.0)) < 1e-6 and abs(pe[0 * 4 + 1, 4] - math.sin(1.0)) < 1e-6
    f = timestep_features(torch.tensor([0.5], dtype=torch.float64), 256)
    assert f.shape == (1, 256)
    assert abs(f[0, 0].item() - math.cos(500.0)) < 1e-3 and abs(f[0, 128].item() - math.sin(500.0)) < 1e-3


def test_unpatchify_order():
    """Output feature f = (p*2 + q)*C + c lands at pixel (2i+p, 2j+q) of channel c."""
    p = init_dit_params(TINY, seed=2)
    H = TINY.hidden
    for b in p["blocks"]:
        b["ada_w"].zero_()
    p["final_ada_w"].zero_()
    p["final_w"].zero_()
    p["final_b"] = torch.arange(16, dtype=torch.float32)
    y = dit_forward(p, torch.zeros(1, 4, 16, 16), torch.zeros(1, dtype=torch.float64),
                    torch.zeros(1, 8, dtype=torch.float64), heads=2)
    for f in range(16):
        c, q, pp = f % 4, (f // 4) % 2, f // 8
        assert y[0, c, pp, q].item() == f
        assert y[0, c, 2 + pp, 4 + q].item() == f


def test_flop_count_convention():
    # DiT-S/2 at 256^2 (256 tokens) is ~6.06 GMAC per the DiT paper; our counter
    # includes attention and embeddings the same way
    s256 = DiTConfig(latent_hw=32)
    assert abs(s256.flops_per_row() / 2e9 - 6.06) < 0.15
    assert abs(DIT_S2.flops_per_row() / 1e9 - 62.86) < 0.5
    assert abs(DIT_XL2.flops_per_row() / 1e9 - 1049.0) < 5.0
