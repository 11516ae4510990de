"""Parity at the shapes the bench runs (BASELINE configs[1]: S=32 streams x n=4 slots =
128 latents = 131072 tokens per step, 256 with CFG).

At these sizes the persistent kernels walk many 128-row tiles per CTA (block tail:
1024 tiles over 148 CTAs), so the cross-tile pipeline phases -- which a <=16-row test
never reaches -- are what runs.  Checks:

* block tail at M = 320 slots x 1024 tokens (2560 row tiles = 1280 CTA-pair tiles over 74
  clusters: 17+ per pair): against the torch-fp32 formula of the block (same tolerance as
  tests/test_gpu_dit_ops.py), and BIT-EXACT against the same kernel run in 8-slot chunks (32
  pair tiles -> one per cluster): a 128-row tile's arithmetic must not depend on which CTA
  pair or pipeline phase computed it;
* DeviceDiT.forward at 128 / 256 rows: bit-identical to 8-row chunks (row independence,
  flowpipe models.py:92-96), first and last chunk against the fp32 oracle on the GPU;
* the bench's own StreamBatch (S=32, device noise, CUDA graph) equal to eager launches
  bit for bit over 6 iterations, with and without CFG.
"""

import numpy as np
import pytest
import torch

from oracle.dit_oracle import dit_forward, params_to

pytestmark = pytest.mark.gpu

T, N, F = 1024, 384, 1536
EPS_TOL_MAX, EPS_TOL_MEAN = 2e-2, 5e-3


def L():
    from paper_2511_22009_b200 import _lib
    return _lib


def st():
    return torch.cuda.current_stream().cuda_stream


def bf(x):
    return x.to(torch.bfloat16)


def _tail_inputs(slots, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    M = slots * T
    d = {
        "attn": bf(torch.randn(M, N, device="cuda", generator=g)),
        "wp": bf(torch.randn(N, N, device="cuda", generator=g) * 0.05),
        "bp": torch.randn(N, device="cuda", generator=g) * 0.1,
        "w1": bf(torch.randn(F, N, device="cuda", generator=g) * 0.05),
        "b1": torch.randn(F, device="cuda", generator=g) * 0.1,
        "w2": bf(torch.randn(N, F, device="cuda", generator=g) * 0.03),
        "b2": torch.randn(N, device="cuda", generator=g) * 0.1,
        "xres0": bf(torch.randn(M, N, device="cuda", generator=g)),
        "vecs": torch.randn(slots, 8 * N, device="cuda", generator=g) * 0.5,
    }
    return d


def _tail(d, xres, xmod, r0, r1):
    """sf_block_tail over slots [r0, r1) (views into the full buffers)."""
    p = lambda t: t.data_ptr()
    v = d["vecs"][r0:]
    vs = 8 * N
    L().call("sf_block_tail", p(d["attn"][r0 * T:]), p(d["wp"]), p(d["bp"]), p(d["w1"]), p(d["w2"]), p(d["b1"]),
             p(d["b2"]), p(xres[r0 * T:]), p(xmod[r0 * T:]), p(v[:, 0:N]), p(v[:, N:]), p(v[:, 2 * N:]),
             p(v[:, 3 * N:]), p(v[:, 4 * N:]), p(v[:, 5 * N:]), vs, 1e-6, (r1 - r0) * T, T, st())


def _tail_ref(d, r0, r1):
    """torch fp32 block tail for slots [r0, r1) (bf16 rounding where the kernel stores bf16)."""
    sl = slice(r0 * T, r1 * T)
    v = d["vecs"][r0:r1].repeat_interleave(T, 0)
    g1, sh1, sc1, g2, sh2, sc2 = (v[:, i * N:(i + 1) * N] for i in range(6))
    ln = lambda x: torch.nn.functional.layer_norm(x, (N,), eps=1e-6)
    x1 = d["xres0"][sl].float() + g1 * (d["attn"][sl].float() @ d["wp"].float().t() + d["bp"])
    h = (ln(x1) * (1 + sc1) + sh1).to(torch.bfloat16).float()
    hh = torch.nn.functional.gelu(h @ d["w1"].float().t() + d["b1"], approximate="tanh").to(torch.bfloat16).float()
    x2 = x1 + g2 * (hh @ d["w2"].float().t() + d["b2"])
    return x2, ln(x2) * (1 + sc2) + sh2


SLOTS = 320  # 2560 row tiles: >= 17 pair tiles per persistent cluster of 2 CTAs
CHUNK = 8    # 64 tiles: one pair tile per cluster


def test_block_tail_multi_tile_bench_shape():
    torch.backends.cuda.matmul.allow_tf32 = False
    d = _tail_inputs(SLOTS, 91)
    M = SLOTS * T
    xres, xmod = d["xres0"].clone(), torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    _tail(d, xres, xmod, 0, SLOTS)
    xres_c, xmod_c = d["xres0"].clone(), torch.empty_like(xmod)
    for r0 in range(0, SLOTS, CHUNK):
        _tail(d, xres_c, xmod_c, r0, r0 + CHUNK)
    torch.cuda.synchronize()
    assert torch.equal(xres, xres_c), "block tail: multi-tile CTAs differ from one-tile CTAs"
    assert torch.equal(xmod, xmod_c), "block tail: multi-tile CTAs differ from one-tile CTAs"
    # formula check on slot ranges at the start, middle and end of the tile walk
    for r0 in (0, 157, SLOTS - 4):
        x2, out = _tail_ref(d, r0, r0 + 4)
        sl = slice(r0 * T, (r0 + 4) * T)
        assert (xres[sl].float() - x2).abs().max().item() < 3e-2 * max(1.0, x2.abs().max().item())
        assert (xmod[sl].float() - out).abs().max().item() < 5e-2 * max(1.0, out.abs().max().item())
    assert torch.isfinite(xmod.float()).all()


@pytest.fixture(scope="module")
def big_dit():
    import paper_2511_22009_b200 as sf
    from paper_2511_22009_b200.dit import DIT_S2

    return sf, sf.DiTVelocityModel(DIT_S2, seed=9, max_rows=256, bias_std=0.02)


@pytest.mark.parametrize("rows", [128, 256])
def test_dit_forward_bench_rows_equal_chunks(big_dit, rows):
    """128 rows (S=32 x n=4) and 256 (with CFG doubling): the whole batch equals the same
    rows run 8 at a time bit for bit; first and last chunk vs the fp32 oracle."""
    _, model = big_dit
    dit = model.device_model
    g = torch.Generator().manual_seed(rows)
    x = torch.randn(rows, 4, 64, 64, generator=g).cuda()
    t = torch.rand(rows, generator=g, dtype=torch.float64).cuda()
    e = torch.randn(rows, 8, generator=g, dtype=torch.float64).cuda()
    full = dit.forward(x, t, e).clone()
    chunks = torch.cat([dit.forward(x[r:r + 8], t[r:r + 8], e[r:r + 8]).clone() for r in range(0, rows, 8)])
    torch.cuda.synchronize()
    assert torch.equal(full, chunks), "DiT forward at bench rows differs from 8-row chunks"
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    pg = params_to(model.params, "cuda")
    for r in (0, rows - 8):
        want = dit_forward(pg, x[r:r + 8], t[r:r + 8], e[r:r + 8], heads=6).reshape(8, -1)
        got = full[r:r + 8]
        scale = want.abs().max().item()
        err = (got - want).abs()
        assert err.max().item() <= EPS_TOL_MAX * scale, (r, err.max().item(), scale)
        assert err.mean().item() <= EPS_TOL_MEAN * scale, (r, err.mean().item(), scale)


@pytest.mark.parametrize("w", [1.0, 7.5])
def test_bench_stream_batch_graph_equals_eager(big_dit, w):
    """bench.py's StreamBatch(S=32, n=4, noise='device', use_graph=True): CUDA-graph replay
    equals eager launches bit for bit over 6 iterations (frames, ids and the whole ring)."""
    sf, model = big_dit
    S, n = 32, 4
    sched = sf.build_time_window_schedule(num_windows=4, inference_steps=n)
    rng = np.random.default_rng(3)
    conds = [sf.make_conditioning(rng.standard_normal(8), guidance_scale=w,
                                  negative_embedding=rng.standard_normal(8) if w != 1.0 else None)
             for _ in range(S)]
    runs = []
    for g in (True, False):
        sb = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=1234, m=None, dtype=np.float32,
                            noise="device", use_graph=g)
        frames = []
        for _ in range(6):
            sb.launch()
            frames.append((sb.frames.clone(), sb.frame_ids.clone()))
        torch.cuda.synchronize()
        runs.append((frames, sb.x_ring.clone()))
        del sb
    (fa, ra), (fb, rb) = runs
    for (xa, ia), (xb, ib) in zip(fa, fb):
        assert torch.equal(ia, ib)
        assert torch.equal(xa, xb)
    assert torch.equal(ra, rb)
    assert torch.isfinite(ra).all()
    assert fa[-1][1].tolist() == [2] * S  # iteration 5 retires generation 5 - 4 + 1 = 2


def test_graph_cache_not_reused_across_batches(big_dit):
    """a StreamBatch freed and re-created with the same shapes must not replay a
    graph that baked in the old one's seed / negative embedding / bookkeeping buffers."""
    sf, model = big_dit
    sched = sf.build_time_window_schedule(num_windows=3, inference_steps=2)
    handle = model.device_model.handle
    outs = {}
    for seed, neg in ((5, None), (6, np.full(8, 0.5)), (6, np.full(8, -1.0))):
        cond = sf.make_conditioning(np.ones(8), guidance_scale=3.0, negative_embedding=neg)
        res = []
        for g in (True, False):
            sb = sf.StreamBatch(model, sched, 2, num_streams=2, cond=cond, seed=seed, m=3, dtype=np.float32,
                                noise="device", use_graph=g)
            res.append(np.stack([r.latent for s in sb() for r in s]))
            del sb
        assert np.array_equal(res[0], res[1]), (seed, neg)
        outs[(seed, None if neg is None else float(neg[0]))] = res[0]
    vals = list(outs.values())
    assert not np.array_equal(vals[0], vals[1]) and not np.array_equal(vals[1], vals[2])
    assert sf._lib.fn("sf_dit_graph_count")(handle) == 0  # every batch released its graphs
