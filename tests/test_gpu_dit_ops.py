"""DiT building blocks on sm_100a vs plain torch fp32 references of the same op:
QKV GEMM with head-major scatter, gated-residual + LayerNorm + modulate
epilogue, tcgen05 flash attention, and the fused block tail."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def L():
    from paper_2511_22009_b200 import _lib
    return _lib


def st():
    return torch.cuda.current_stream().cuda_stream


def bf(x):
    return x.to(torch.bfloat16)


@pytest.mark.parametrize("rows", [1, 3])
def test_qkv_scatter(rows):
    T, H = 1024, 6
    d = H * 64
    M = rows * T
    g = torch.Generator(device="cuda").manual_seed(rows)
    a = bf(torch.randn(M, d, device="cuda", generator=g))
    w = bf(torch.randn(3 * d, d, device="cuda", generator=g) * 0.05)
    b = torch.randn(3 * d, device="cuda", generator=g) * 0.1
    q = torch.empty(rows, H, T, 64, device="cuda", dtype=torch.bfloat16)
    k = torch.empty_like(q)
    vt = torch.empty(rows, H, 64, T, device="cuda", dtype=torch.float16)
    L().call("sf_gemm_qkv", a.data_ptr(), w.data_ptr(), b.data_ptr(), q.data_ptr(), k.data_ptr(),
             vt.data_ptr(), M, H, T, 0.125, st())
    torch.cuda.synchronize()
    ref = (a.float() @ w.float().t() + b).view(rows, T, 3, H, 64)
    rq = ref[:, :, 0].permute(0, 2, 1, 3) * 0.125
    rk = ref[:, :, 1].permute(0, 2, 1, 3)
    rv = ref[:, :, 2].permute(0, 2, 3, 1)
    for got, want in ((q, rq), (k, rk), (vt, rv)):
        assert (got.float() - want).abs().max().item() < 2e-2 * max(1.0, want.abs().max().item())


@pytest.mark.parametrize("K,rows", [(384, 2), (1536, 2), (1536, 1), (1536, 3)])
def test_res_ln_epilogue(K, rows):
    T, N = 1024, 384
    M = rows * T
    g = torch.Generator(device="cuda").manual_seed(K)
    a = bf(torch.randn(M, K, device="cuda", generator=g))
    w = bf(torch.randn(N, K, device="cuda", generator=g) * 0.05)
    b = torch.randn(N, device="cuda", generator=g) * 0.1
    xres = bf(torch.randn(M, N, device="cuda", generator=g))
    x0 = xres.float().clone()
    vec_stride = 4 * N
    vecs = torch.randn(rows, vec_stride, device="cuda", generator=g) * 0.5
    gate, shift, scale = vecs[:, 0:N], vecs[:, N:2 * N], vecs[:, 2 * N:3 * N]
    xmod = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    L().call("sf_gemm_res_ln", a.data_ptr(), w.data_ptr(), b.data_ptr(), xres.data_ptr(),
             xmod.data_ptr(), gate.data_ptr(), shift.data_ptr(), scale.data_ptr(), vec_stride,
             M, N, K, T, 1e-6, st())
    torch.cuda.synchronize()
    slot = torch.arange(M, device="cuda") // T
    y = x0 + gate[slot] * (a.float() @ w.float().t() + b)
    assert (xres.float() - y).abs().max().item() < 3e-2 * max(1.0, y.abs().max().item())
    ln = torch.nn.functional.layer_norm(y, (N,), eps=1e-6)
    ref = ln * (1 + scale[slot]) + shift[slot]
    assert (xmod.float() - ref).abs().max().item() < 5e-2 * max(1.0, ref.abs().max().item())


@pytest.mark.parametrize("rows,H,scale", [(1, 6, 1.0), (2, 6, 4.0), (1, 16, 8.0)])
def test_attention_matches_sdpa(rows, H, scale):
    T = 1024
    g = torch.Generator(device="cuda").manual_seed(rows * H)
    q = bf(torch.randn(rows, H, T, 64, device="cuda", generator=g) * scale / 8)
    k = bf(torch.randn(rows, H, T, 64, device="cuda", generator=g))
    v = bf(torch.randn(rows, H, T, 64, device="cuda", generator=g))
    vt = v.transpose(-1, -2).contiguous().to(torch.float16)  # PV runs in fp16
    out = torch.empty(rows * T, H * 64, device="cuda", dtype=torch.bfloat16)
    L().call("sf_attention", q.data_ptr(), k.data_ptr(), vt.data_ptr(), out.data_ptr(), rows, H, T, st())
    torch.cuda.synchronize()
    # q already carries the 1/sqrt(d) factor -> sdpa with scale=1
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float(), scale=1.0)
    ref = ref.permute(0, 2, 1, 3).reshape(rows * T, H * 64)
    err = (out.float() - ref).abs().max().item()
    assert err < 2e-2, err


@pytest.mark.parametrize("rows,H,scale", [(1, 16, 1.0), (2, 16, 6.0)])
def test_attention_hd72_matches_sdpa(rows, H, scale):
    """Head dim 72 (DiT-XL/2): QK^T zero-padded to 80 on chip, ones-row at 72."""
    T, hd = 1024, 72
    g = torch.Generator(device="cuda").manual_seed(7 + rows)
    q = bf(torch.randn(rows, H, T, hd, device="cuda", generator=g) * scale / hd ** 0.5)
    k = bf(torch.randn(rows, H, T, hd, device="cuda", generator=g))
    v = bf(torch.randn(rows, H, T, hd, device="cuda", generator=g))
    vt = v.transpose(-1, -2).contiguous().to(torch.float16)
    out = torch.empty(rows * T, H * hd, device="cuda", dtype=torch.bfloat16)
    L().call("sf_attention_hd", q.data_ptr(), k.data_ptr(), vt.data_ptr(), out.data_ptr(), rows, H, T, hd, st())
    torch.cuda.synchronize()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float(), scale=1.0)
    ref = ref.permute(0, 2, 1, 3).reshape(rows * T, H * hd)
    err = (out.float() - ref).abs().max().item()
    assert err < 2e-2, err


@pytest.mark.parametrize("rows", [2, 4])
def test_block_tail_matches_gemm_path(rows):
    """sf_block_tail (projection + residual + LN + MLP + residual + LN in one kernel on CTA pairs)
    vs the GEMM path sf_gemm_res_ln (projection) -> sf_gemm_bf16 GELU (fc1) -> sf_gemm_res_ln
    (fc2), and vs torch fp32."""
    T, N, F = 1024, 384, 1536
    M = rows * T
    g = torch.Generator(device="cuda").manual_seed(70 + rows)
    attn = bf(torch.randn(M, N, device="cuda", generator=g))
    wp = bf(torch.randn(N, N, device="cuda", generator=g) * 0.05)
    bp = torch.randn(N, device="cuda", generator=g) * 0.1
    w1 = bf(torch.randn(F, N, device="cuda", generator=g) * 0.05)
    b1 = torch.randn(F, device="cuda", generator=g) * 0.1
    w2 = bf(torch.randn(N, F, device="cuda", generator=g) * 0.03)
    b2 = torch.randn(N, device="cuda", generator=g) * 0.1
    xres0 = bf(torch.randn(M, N, device="cuda", generator=g))
    vs = 8 * N
    vecs = torch.randn(rows, vs, device="cuda", generator=g) * 0.5
    g1, sh1, sc1 = vecs[:, 0:N], vecs[:, N:2 * N], vecs[:, 2 * N:3 * N]
    g2, sh2, sc2 = vecs[:, 3 * N:4 * N], vecs[:, 4 * N:5 * N], vecs[:, 5 * N:6 * N]
    ptr = lambda t: t.data_ptr()
    # one kernel
    xres = xres0.clone()
    xmod = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    L().call("sf_block_tail", ptr(attn), ptr(wp), ptr(bp), ptr(w1), ptr(w2), ptr(b1), ptr(b2), ptr(xres), ptr(xmod),
             ptr(g1), ptr(sh1), ptr(sc1), ptr(g2), ptr(sh2), ptr(sc2), vs, 1e-6, M, T, st())
    # three GEMMs
    xres_u = xres0.clone()
    h_u = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    hid = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    xmod_u = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    L().call("sf_gemm_res_ln", ptr(attn), ptr(wp), ptr(bp), ptr(xres_u), ptr(h_u), ptr(g1), ptr(sh1), ptr(sc1),
             vs, M, N, N, T, 1e-6, st())
    L().call("sf_gemm_bf16", ptr(h_u), ptr(w1), ptr(b1), ptr(hid), M, F, N, 2, st())
    L().call("sf_gemm_res_ln", ptr(hid), ptr(w2), ptr(b2), ptr(xres_u), ptr(xmod_u), ptr(g2), ptr(sh2), ptr(sc2),
             vs, M, N, F, T, 1e-6, st())
    torch.cuda.synchronize()
    slot = torch.arange(M, device="cuda") // T
    ln = lambda x: torch.nn.functional.layer_norm(x, (N,), eps=1e-6)
    x1 = xres0.float() + g1[slot] * (attn.float() @ wp.float().t() + bp)
    h = (ln(x1) * (1 + sc1[slot]) + sh1[slot]).to(torch.bfloat16).float()
    hh = torch.nn.functional.gelu(h @ w1.float().t() + b1, approximate="tanh").to(torch.bfloat16).float()
    x2 = x1 + g2[slot] * (hh @ w2.float().t() + b2)
    out = ln(x2) * (1 + sc2[slot]) + sh2[slot]
    for r, m in ((xres, xmod), (xres_u, xmod_u)):
        assert (r.float() - x2).abs().max().item() < 3e-2 * max(1.0, x2.abs().max().item())
        assert (m.float() - out).abs().max().item() < 5e-2 * max(1.0, out.abs().max().item())
    assert (xres.float() - xres_u.float()).abs().max().item() < 2e-2 * max(1.0, x2.abs().max().item())


def test_block_tail_rejects_bad_shapes():
    """sf_block_tail refuses row counts that are not whole pairs of 128-row tiles of whole slots,
    and null pointers (ParameterError, like the reference's shape checks)."""
    from paper_2511_22009_b200.errors import ParameterError

    N, F = 384, 1536
    z = torch.zeros(256, N, device="cuda", dtype=torch.bfloat16)
    w1 = torch.zeros(F, N, device="cuda", dtype=torch.bfloat16)
    w2 = torch.zeros(N, F, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(F, device="cuda")
    v = torch.zeros(1, 8 * N, device="cuda")
    args = lambda a0, M, T: (a0, z.data_ptr(), b.data_ptr(), w1.data_ptr(), w2.data_ptr(), b.data_ptr(), b.data_ptr(),
                             z.data_ptr(), z.data_ptr(), *([v.data_ptr()] * 6), 8 * N, 1e-6, M, T, st())
    with pytest.raises(ParameterError):  # M not a multiple of 256 (one 128-row tile)
        L().call("sf_block_tail", *args(z.data_ptr(), 128, 128))
    with pytest.raises(ParameterError):  # tokens per slot not a multiple of 128
        L().call("sf_block_tail", *args(z.data_ptr(), 256, 100))
    with pytest.raises(ParameterError):  # null pointer
        L().call("sf_block_tail", *args(None, 256, 128))
