"""Stream partitioning across ranks.

Streams are independent run_stream invocations (reference SPEC: independent
runs share nothing), so S_total streams are split into contiguous blocks, one
per rank, with no collective inside the step.  Global stream g keeps the run
seed ``base_seed + g`` wherever it runs, so an N-GPU run produces exactly the
frames of a 1-GPU run over the same S_total streams.  NCCL (or gloo on CPU) is
used only off the hot loop, to gather emitted frames and counters.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def stream_partition(total_streams: int, world: int, rank: int) -> range:
    """Contiguous block of global stream ids owned by `rank` (remainder to the
    lowest ranks)."""
    if total_streams < 1 or world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad partition request ({total_streams}, {world}, {rank})")
    base, rem = divmod(total_streams, world)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


def stream_seeds(base_seed: int, streams: range) -> list[int]:
    return [base_seed + g for g in streams]


def gather_frames(frames: torch.Tensor, frame_ids: torch.Tensor, group=None):
    """All-gather every rank's emitted frames [S_local, D] and ids [S_local]
    (ragged S_local allowed) -> ([S_total, D], [S_total]) in global stream order."""
    world = dist.get_world_size(group)
    n_local = torch.tensor([frames.shape[0]], device=frames.device, dtype=torch.int64)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    pad = torch.zeros(mx, frames.shape[1], dtype=frames.dtype, device=frames.device)
    pad[: frames.shape[0]] = frames
    ipad = torch.full((mx,), -1, dtype=torch.int64, device=frames.device)
    ipad[: frame_ids.shape[0]] = frame_ids
    outs = [torch.empty_like(pad) for _ in range(world)]
    ids = [torch.empty_like(ipad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    dist.all_gather(ids, ipad, group=group)
    return (torch.cat([o[:s] for o, s in zip(outs, sizes)]), torch.cat([i[:s] for i, s in zip(ids, sizes)]))


def reduce_counts(counts: list[int], device, group=None) -> list[int]:
    """Sum integer counters (frames, model calls, param evals, ...) over ranks."""
    t = torch.tensor(counts, dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    return [int(v) for v in t.tolist()]
