"""DiT stream batch on the GPU vs the oracle stream loop driving the torch-fp32
CPU DiT (oracle/dit_oracle.py + oracle/flowpipe_oracle.py).

Queue order, ids, stages and counters are exact.  Latent trajectories (fp32
state, bf16 network): max |x_gpu - x_cpu| / max |x_cpu| <= 1e-2.
"""

import numpy as np
import pytest
import torch

from oracle import flowpipe_oracle as O
from oracle.dit_oracle import dit_forward

pytestmark = pytest.mark.gpu
TRAJ_TOL = 1e-2


@pytest.fixture(scope="module")
def setup():
    import paper_2511_22009_b200 as sf
    from paper_2511_22009_b200.dit import DIT_S2

    model = sf.DiTVelocityModel(DIT_S2, seed=5, max_rows=16, bias_std=0.02)
    return sf, model


@pytest.mark.parametrize("k,w", [(3, 1.0), (4, 4.0)])
def test_dit_stream_matches_cpu_oracle(setup, k, w):
    sf, model = setup
    S, m, n, D = 2, 3, 4, model.dim
    sched = sf.build_time_window_schedule(num_windows=k, inference_steps=n)
    rng = np.random.default_rng(1)
    embs = [rng.standard_normal(8) for _ in range(S)]
    conds = [sf.make_conditioning(embs[s], guidance_scale=w) for s in range(S)]
    sb = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=50, m=m, dtype=np.float32)
    out = sb()
    osch = O.make_schedule(num_windows=k, steps=n)
    for s in range(S):
        def eps_fn(ids, ts, x, s=s):
            B = len(ids)
            xt = torch.from_numpy(np.asarray(x, np.float32)).view(B, 4, 64, 64)
            tt = torch.as_tensor(ts, dtype=torch.float64)
            ec = torch.as_tensor(np.tile(embs[s], (B, 1)))
            e_c = dit_forward(model.params, xt, tt, ec, heads=6).reshape(B, D)
            if w == 1.0:
                return e_c.numpy()
            e_u = dit_forward(model.params, xt, tt, torch.zeros_like(ec), heads=6).reshape(B, D)
            return (e_u + w * (e_c - e_u)).numpy()
        run = O.run_stream(m, n, eps_fn, 50 + s, osch, D, dtype=np.float32)
        assert [r.id for r in out[s]] == run.order
        # the CFG combine amplifies the network's error by |w| + |w - 1| = 2w - 1
        tol = TRAJ_TOL * max(1.0, (2 * w - 1) / 3)
        for r in out[s]:
            want = run.latents[r.id]
            err = np.abs(r.latent - want).max() / np.abs(want).max()
            print(f"K={k} w={w} stream {s} gen {r.id}: normalised max err {err:.2e} (tol {tol:.1e})")
            assert err <= tol, (s, r.id, err)
        assert sb.stats[s].model_calls == m + n - 1
        assert sb.stats[s].step_stats.param_evals == m * n


def test_graph_replay_equals_eager(setup):
    sf, model = setup
    sched = sf.build_time_window_schedule(num_windows=3, inference_steps=4)
    cond = sf.make_conditioning(np.ones(8), guidance_scale=2.0)
    outs = []
    for g in (True, False):
        sb = sf.StreamBatch(model, sched, 4, num_streams=2, cond=cond, seed=7, m=5, dtype=np.float32,
                            noise="device", use_graph=g)
        outs.append(sb())
    for a, b in zip(outs[0], outs[1]):
        for ra, rb in zip(a, b):
            assert ra.id == rb.id and np.array_equal(ra.latent, rb.latent)


def _oracle_eps_gpu(params_gpu, emb, neg, w, heads):
    """Guided eps of the fp32 DiT reference run on the GPU (TF32 off), in the reference's
    CFG layout: [uncond (neg or zeros) ; cond] combined as e_u + w (e_c - e_u)
    (models.py:257-268, :288-293)."""
    def eps_fn(ids, ts, x):
        B = len(ids)
        xt = torch.from_numpy(np.asarray(x, np.float32)).view(B, 4, 64, 64).cuda()
        tt = torch.as_tensor(ts, dtype=torch.float64).cuda()
        ec = torch.as_tensor(np.tile(emb, (B, 1))).cuda()
        e_c = dit_forward(params_gpu, xt, tt, ec, heads=heads).reshape(B, -1)
        if w == 1.0:
            return e_c.cpu().numpy()
        en = torch.zeros_like(ec) if neg is None else torch.as_tensor(np.tile(neg, (B, 1))).cuda()
        e_u = dit_forward(params_gpu, xt, tt, en, heads=heads).reshape(B, -1)
        return (e_u + w * (e_c - e_u)).cpu().numpy()
    return eps_fn


@pytest.mark.parametrize("n", [1, 2])
def test_dit_cfg_negative_embedding_short_grids(setup, n):
    """configs[2]: CFG (w=7.5) with a NON-ZERO negative embedding on 1- and 2-step grids,
    through the fused stream step (the fused kernel's neg pointer), vs the oracle loop."""
    from oracle.dit_oracle import params_to

    sf, model = setup
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    S, m, w, D = 2, 3, 7.5, model.dim
    sched = sf.build_time_window_schedule(num_windows=4, inference_steps=n)
    rng = np.random.default_rng(20 + n)
    embs = [rng.standard_normal(8) for _ in range(S)]
    negs = [rng.standard_normal(8) for _ in range(S)]
    conds = [sf.make_conditioning(embs[s], guidance_scale=w, negative_embedding=negs[s]) for s in range(S)]
    sb = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=70, m=m, dtype=np.float32)
    out = sb()
    osch = O.make_schedule(num_windows=4, steps=n)
    pg = params_to(model.params, "cuda")
    tol = TRAJ_TOL * max(1.0, (2 * w - 1) / 3)
    for s in range(S):
        run = O.run_stream(m, n, _oracle_eps_gpu(pg, embs[s], negs[s], w, 6), 70 + s, osch, D, dtype=np.float32)
        assert [r.id for r in out[s]] == run.order
        for r in out[s]:
            want = run.latents[r.id]
            err = np.abs(r.latent - want).max() / np.abs(want).max()
            print(f"n={n} stream {s} gen {r.id}: normalised max err {err:.2e} (tol {tol:.1e})")
            assert err <= tol, (s, r.id, err)
        assert sb.stats[s].model_calls == m + n - 1
    # the negative embedding matters: the zero-negative run differs
    conds0 = [sf.make_conditioning(embs[s], guidance_scale=w) for s in range(S)]
    out0 = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds0, seed=70, m=m, dtype=np.float32)()
    assert not np.array_equal(out0[0][0].latent, out[0][0].latent)


def test_dit_xl_stream_step_matches_oracle():
    """configs[3]: the DiT-XL/2 fused stream step (final layer <1152> in stream mode,
    hd-72 attention, RES + LayerNorm pass) over an 8-slot batch (S=2 x n=4) vs the oracle
    loop driving the fp32 XL reference on the GPU.  Tolerance: the XL forward bound (3e-2,
    tests/test_gpu_dit_xl.py) carried through the trajectory."""
    import paper_2511_22009_b200 as sf
    from oracle.dit_oracle import params_to
    from paper_2511_22009_b200.dit import DIT_XL2

    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    model = sf.DiTVelocityModel(DIT_XL2, seed=4, max_rows=8, bias_std=0.02)
    S, m, n, D = 2, 2, 4, model.dim
    sched = sf.build_time_window_schedule(num_windows=3, inference_steps=n)
    rng = np.random.default_rng(8)
    embs = [rng.standard_normal(8) for _ in range(S)]
    conds = [sf.make_conditioning(embs[s]) for s in range(S)]
    sb = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=90, m=m, dtype=np.float32)
    out = sb()
    osch = O.make_schedule(num_windows=3, steps=n)
    pg = params_to(model.params, "cuda")
    for s in range(S):
        run = O.run_stream(m, n, _oracle_eps_gpu(pg, embs[s], None, 1.0, 16), 90 + s, osch, D, dtype=np.float32)
        assert [r.id for r in out[s]] == run.order
        for r in out[s]:
            want = run.latents[r.id]
            err = np.abs(r.latent - want).max() / np.abs(want).max()
            print(f"XL stream {s} gen {r.id}: normalised max err {err:.2e}")
            assert err <= 3 * TRAJ_TOL, (s, r.id, err)


def test_dit_mixed_guidance_equals_separate_batches(setup):
    """Per-stream guidance scales in one DiT stream batch (CFG rows for every stream, each combined
    with its own w; w == 1 streams take the conditional eps) == each stream run alone, bit for bit
    (row independence of the network)."""
    sf, model = setup
    n, m = 2, 3
    sched = sf.build_time_window_schedule(num_windows=3, inference_steps=n)
    rng = np.random.default_rng(12)
    embs = [rng.standard_normal(8) for _ in range(2)]
    ws = [1.0, 5.0]
    conds = [sf.make_conditioning(embs[s], guidance_scale=ws[s]) for s in range(2)]
    mixed = sf.StreamBatch(model, sched, n, num_streams=2, cond=conds, seed=[40, 41], m=m, dtype=np.float32)()
    for s in range(2):
        alone = sf.StreamBatch(model, sched, n, num_streams=1, cond=conds[s], seed=40 + s, m=m, dtype=np.float32)()
        for a, b in zip(mixed[s], alone[0]):
            assert a.id == b.id and np.array_equal(a.latent, b.latent), (s, a.id)


@pytest.mark.parametrize("w", [1.0, 3.0])
def test_device_noise_refill_equals_philox_fill(setup, w):
    """noise='device': the final-layer kernel draws the admitted generation's noise itself (Philox
    counters shared across lanes); the admitted ring rows must equal sf_philox_normal's output for
    (seeds[0] + s, generation j + 1) element for element, with and without the CFG tile pair."""
    sf, model = setup
    from paper_2511_22009_b200 import _lib

    S, n = 2, 4  # 16 network rows with CFG (the fixture's max_rows)
    sched = sf.build_time_window_schedule(num_windows=3, inference_steps=n)
    cond = sf.make_conditioning(np.ones(8), guidance_scale=w)
    sb = sf.StreamBatch(model, sched, n, num_streams=S, cond=cond, seed=11, m=6, dtype=np.float32,
                        noise="device", use_graph=False)
    st = torch.cuda.current_stream().cuda_stream
    ref = torch.empty(S, model.dim, dtype=torch.float32, device="cuda")
    _lib.call("sf_philox_normal", ref.data_ptr(), S, model.dim, sb.noise_seed, 0, st)
    ring = sb.x_ring.view(S, n, -1)
    assert torch.equal(ring[:, 0], ref)  # generation 0 (reset)
    for j in range(3):
        sb.launch()
        _lib.call("sf_philox_normal", ref.data_ptr(), S, model.dim, sb.noise_seed, j + 1, st)
        torch.cuda.synchronize()
        assert torch.equal(ring[:, (j + 1) % n], ref), j


def test_launch_host_io_overlapped_copies_match_launch(setup):
    """launch_host_io (H2D of the admission noise and D2H of the frames on a side stream, double-
    buffered device noise / frames) gives the same frames as uploading the same noise and calling
    launch() on the current stream, step for step (graph replay, 7 steps: both buffers reused)."""
    sf, model = setup
    S, n = 2, 4
    sched = sf.build_time_window_schedule(num_windows=3, inference_steps=n)
    cond = sf.make_conditioning(np.ones(8), guidance_scale=1.0)
    mk = lambda: sf.StreamBatch(model, sched, n, num_streams=S, cond=cond, seed=21, dtype=np.float32, noise="host")
    a, b = mk(), mk()
    g = torch.Generator().manual_seed(4)
    noises = [torch.randn(S, model.dim, generator=g).pin_memory() for _ in range(7)]
    dsts = [torch.empty(S, model.dim).pin_memory() for _ in range(7)]
    for j in range(7):
        a.noise_dev.copy_(noises[j].cuda())
        a.launch()
        want = a.frames.cpu()
        b.launch_host_io(noises[j], dsts[j])
        b.io_join()
        torch.cuda.synchronize()
        assert torch.equal(a.frame_ids, b.frame_ids), j
        ok = (a.frame_ids >= 0).cpu()  # streams that retired a frame this step
        assert torch.equal(dsts[j][ok], want[ok]), j
        assert torch.equal(b.frames.cpu()[ok], want[ok]), j
    assert ok.all()  # steady state reached


def test_batch_of_streams_equals_single_stream_batches():
    """One DiT StreamBatch of 5 streams (20 network rows: plain launches) gives every stream the
    frames of its own single-stream batch (4 rows: the small-batch programmatic-dependent-launch
    path), bit for bit: row independence across batch sizes and launch modes."""
    import paper_2511_22009_b200 as sf
    from paper_2511_22009_b200.dit import DIT_S2

    model = sf.DiTVelocityModel(DIT_S2, seed=9, max_rows=20, bias_std=0.02)
    S, n, m = 5, 4, 6
    sched = sf.build_time_window_schedule(num_windows=4, inference_steps=n)
    rng = np.random.default_rng(3)
    conds = [sf.make_conditioning(rng.standard_normal(8)) for _ in range(S)]
    seeds = [100 + 7 * s for s in range(S)]
    big = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=seeds, m=m, dtype=np.float32)()
    for s in range(S):
        one = sf.StreamBatch(model, sched, n, num_streams=1, cond=[conds[s]], seed=[seeds[s]], m=m,
                             dtype=np.float32)()[0]
        assert [r.id for r in one] == [r.id for r in big[s]]
        for a, b in zip(one, big[s]):
            assert np.array_equal(a.latent, b.latent), (s, a.id)


@pytest.mark.parametrize("S,n,m", [(3, 2, 4), (6, 4, 5)])
def test_batch_of_guided_streams_equals_single_stream_batches(S, n, m):
    """Per-stream guidance scales (1.0 included) with and without negative embeddings: one guided
    DiT batch (2 S n network rows: 12 rows = the small-batch PDL path, 48 rows = plain launches)
    gives each stream the frames of its own single-stream batch, bit for bit."""
    import paper_2511_22009_b200 as sf
    from paper_2511_22009_b200.dit import DIT_S2

    model = sf.DiTVelocityModel(DIT_S2, seed=5, max_rows=2 * S * n, bias_std=0.02)
    sched = sf.build_time_window_schedule(num_windows=3, inference_steps=n)
    rng = np.random.default_rng(S * 10 + n)
    ws = [1.0, 4.0, 7.5, 2.5, 1.0, 6.0][:S]
    conds = [sf.make_conditioning(rng.standard_normal(8), guidance_scale=ws[s],
                                  negative_embedding=rng.standard_normal(8) if s % 2 else None) for s in range(S)]
    seeds = [int(v) for v in rng.integers(0, 2**31, size=S)]
    big = sf.StreamBatch(model, sched, n, num_streams=S, cond=conds, seed=seeds, m=m, dtype=np.float32)()
    for s in range(S):
        one = sf.StreamBatch(model, sched, n, num_streams=1, cond=[conds[s]], seed=[seeds[s]], m=m,
                             dtype=np.float32)()[0]
        assert [r.id for r in one] == [r.id for r in big[s]]
        for a, b in zip(one, big[s]):
            assert np.array_equal(a.latent, b.latent), (s, a.id)


def test_finalizer_order_model_before_batch():
    """A DiT StreamBatch and its model collected in either order (as a garbage cycle at interpreter
    shutdown may do): the model's finalizer destroys the runtime handle and nulls it, so the
    batch's finalizer, run afterwards, sees NULL instead of a freed handle, and the model's own
    finalizer running again is a no-op (subprocess: a use-after-free would kill the interpreter)."""
    import subprocess
    import sys

    code = r'''
import numpy as np, torch
import paper_2511_22009_b200 as sf
from paper_2511_22009_b200.dit import DIT_S2
model = sf.DiTVelocityModel(DIT_S2, seed=1, max_rows=8)
sched = sf.build_time_window_schedule(inference_steps=4)
sb = sf.StreamBatch(model, sched, 4, num_streams=2, cond=sf.make_conditioning(np.ones(8)), seed=0,
                    dtype=np.float32, noise="device", use_graph=True)
for _ in range(3):
    sb.launch()
torch.cuda.synchronize()
dm = model.device_model
dm.__del__()      # the model first ...
sb.__del__()      # ... then the batch's graph release: must see a NULL handle
dm.__del__()      # and a second finalizer call must not destroy again
del sb, model, dm
import gc; gc.collect()
print("finalizers ok")
'''
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "finalizers ok" in r.stdout, (r.returncode, r.stdout[-500:], r.stderr[-2000:])
