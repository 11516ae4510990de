"""Multi-rank correctness of the stream partition (reference SPEC.md:334:
independent runs share nothing) without an 8-GPU node: two processes on cuda:0, gloo over
host-staged tensors.  Each rank runs a StreamBatch over ``stream_partition(S_total, 2, r)``
with ``stream_seeds``, records every step's frames (partition.FrameWindow) and gathers
them once at the end; the gathered frames, in global stream order, must equal ONE
StreamBatch over all S_total streams bit for bit -- for the mock model (fp64) and the
DiT (fp32 ring, bf16 network), with numpy-identical and Philox admission noise."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

S_TOTAL, N, M, SEED = 5, 4, 6, 300


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _batch(kind, noise, streams, seeds):
    import paper_2511_22009_b200 as sf
    from paper_2511_22009_b200.dit import DIT_S2

    sched = sf.build_time_window_schedule(num_windows=3, inference_steps=N)
    conds = [sf.make_conditioning(np.random.default_rng([sd, 2**32 - 1]).standard_normal(8), guidance_scale=2.5)
             for sd in seeds]
    if kind == "mock":
        model, dt = sf.SeededMockModel(dim=4096, seed=17), np.float64
    else:
        model, dt = sf.DiTVelocityModel(DIT_S2, seed=21, max_rows=2 * S_TOTAL * N, bias_std=0.02), np.float32
    return sf.StreamBatch(model, sched, N, num_streams=len(streams), cond=conds, seed=seeds, m=M, dtype=dt,
                          noise=noise)


def _run(sb, window):
    frames = []
    while not sb.done():
        sb.launch()
        if window is not None:
            window.record()
        else:
            frames.append((sb.frames.clone(), sb.frame_ids.clone()))
    return frames


def _rank(rank, world, port, kind, noise, q):
    import torch.distributed as dist

    from paper_2511_22009_b200.partition import FrameWindow, stream_partition, stream_seeds

    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = stream_partition(S_TOTAL, world, rank)
    sb = _batch(kind, noise, mine, stream_seeds(SEED, mine))
    fw = FrameWindow(sb, window=M + N - 1)
    _run(sb, fw)
    f, ids = fw.gather()
    if rank == 0:
        q.put((f.cpu().numpy(), ids.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,noise", [("mock", "numpy"), ("dit", "numpy"), ("dit", "device")])
def test_two_ranks_equal_one_rank(kind, noise):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, kind, noise, q)) for r in range(2)]
    for p in procs:
        p.start()
    frames, ids = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # one rank, all streams
    sb = _batch(kind, noise, range(S_TOTAL), [SEED + g for g in range(S_TOTAL)])
    ref = _run(sb, None)
    assert frames.shape[0] == len(ref) == M + N - 1 and frames.shape[1] == S_TOTAL
    for k, (rf, ri) in enumerate(ref):
        assert np.array_equal(ids[k], ri.cpu().numpy()), k
        assert np.array_equal(frames[k], rf.cpu().numpy()), (kind, noise, k)
    emitted = ids[ids >= 0]
    assert len(emitted) == M * S_TOTAL  # every generation of every stream, once
