"""Multi-rank host logic on CPU (gloo, world_size 2): stream partitioning and
the off-hot-loop gather of frames / counters that bench.py runs over NCCL."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_22009_b200.partition import gather_frames, reduce_counts, stream_partition, stream_seeds


def test_partition_is_a_disjoint_cover():
    for total in (1, 5, 64, 513):
        for world in (1, 2, 3, 8):
            if world > total:
                continue
            got = [g for r in range(world) for g in stream_partition(total, world, r)]
            assert got == list(range(total))
            sizes = [len(stream_partition(total, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    assert stream_seeds(1000, range(3, 6)) == [1003, 1004, 1005]
    with pytest.raises(ValueError):
        stream_partition(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, D, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = stream_partition(total, world, rank)
    # each stream's "frame" is a deterministic function of its global id
    frames = torch.stack([torch.full((D,), float(g)) for g in mine]) if len(mine) else torch.zeros(0, D)
    ids = torch.tensor(list(mine), dtype=torch.int64)
    allf, allid = gather_frames(frames, ids)
    counts = reduce_counts([len(mine), 10 * (rank + 1)], "cpu")
    if rank == 0:
        q.put((allf.numpy().tolist(), allid.tolist(), counts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [4, 5])
def test_gather_frames_world2(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    D = 6
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, D, q)) for r in range(2)]
    for p in procs:
        p.start()
    frames, ids, counts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ids == list(range(total))
    for g, row in enumerate(frames):
        assert row == [float(g)] * D
    assert counts == [total, 30]


def _window_worker(rank, world, port, total, D, steps, q):
    """CPU stand-in for a StreamBatch: frame of (stream g, step k) = g * 100 + k."""
    from paper_2511_22009_b200.partition import FrameWindow

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = stream_partition(total, world, rank)

    class FakeBatch:
        frames = torch.zeros(len(mine), D)
        frame_ids = torch.zeros(len(mine), dtype=torch.int64)

    fw = FrameWindow(FakeBatch, window=steps)
    for k in range(steps):
        FakeBatch.frames.copy_(torch.tensor([[g * 100.0 + k] * D for g in mine]))
        FakeBatch.frame_ids.fill_(k - 1)
        fw.record()
    f, ids = fw.gather()
    if rank == 0:
        q.put((f.numpy().tolist(), ids.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_frame_window_gathers_every_step_world2():
    """FrameWindow: every step's frames of every rank, in (step, global stream) order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    total, D, steps = 5, 3, 4
    procs = [ctx.Process(target=_window_worker, args=(r, 2, port, total, D, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    frames, ids = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(frames) == steps and all(len(f) == total for f in frames)
    for k in range(steps):
        assert ids[k] == [k - 1] * total
        for g in range(total):
            assert frames[k][g] == [g * 100.0 + k] * D
