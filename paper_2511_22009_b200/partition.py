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


def all_gather_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather a [n_local, ...] tensor with ragged n_local across ranks -> [n_total, ...]
    in rank order (sizes exchanged first, rows padded to the largest rank)."""
    world = dist.get_world_size(group)
    n_local = torch.tensor([t.shape[0]], device=t.device, dtype=torch.int64)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(s.item()) for s in sizes]
    pad = torch.zeros((max(sizes),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:s] for o, s in zip(outs, sizes)])


def gather_frames(frames: torch.Tensor, frame_ids: torch.Tensor, group=None):
    """All-gather every rank's emitted frames [S_local, D] and ids [S_local]
    (ragged S_local allowed) -> ([S_total, D], [S_total]) in global stream order."""
    return all_gather_rows(frames, group), all_gather_rows(frame_ids, group)


def _staged(t: torch.Tensor, group=None) -> torch.Tensor:
    """gloo moves CPU tensors: stage device tensors through the host for it."""
    return t.cpu() if t.is_cuda and dist.get_backend(group) == "gloo" else t


class FrameWindow:
    """Every frame a rank's StreamBatch emits, collected on the device step by step and
    gathered across ranks once per window (no collective inside the step).

    ``record()`` after each ``StreamBatch.launch()`` copies that step's frames [S_local, D]
    and generation ids into slot i of a device buffer [window, S_local, D] (stream-ordered,
    no host sync); ``gather()`` all-gathers the filled slots -> ([steps, S_total, D],
    [steps, S_total]) in global stream order on every rank, and restarts the window."""

    def __init__(self, sb, window: int, group=None):
        if window < 1:
            raise ValueError("window must be >= 1")
        self.sb, self.window, self.group = sb, int(window), group
        S, D = sb.frames.shape
        self.frames = torch.zeros(self.window, S, D, dtype=sb.frames.dtype, device=sb.frames.device)
        self.ids = torch.full((self.window, S), -1, dtype=torch.int64, device=sb.frames.device)
        self.n = 0

    def record(self) -> None:
        if self.n >= self.window:
            raise RuntimeError("frame window full: gather() it first")
        self.frames[self.n].copy_(self.sb.frames, non_blocking=True)
        self.ids[self.n].copy_(self.sb.frame_ids, non_blocking=True)
        self.n += 1

    def gather(self):
        w = self.n
        f = self.frames[:w].transpose(0, 1).contiguous()  # [S_local, w, D]: rows = local streams
        i = self.ids[:w].t().contiguous()
        allf = all_gather_rows(_staged(f, self.group), self.group)
        alli = all_gather_rows(_staged(i, self.group), self.group)
        self.n = 0
        return allf.transpose(0, 1).contiguous(), alli.t().contiguous()


def reduce_counts(counts: list[int], device, group=None) -> list[int]:
    """Sum integer counters (frames, model calls, param evals, ...) over ranks."""
    t = torch.tensor(counts, dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    return [int(v) for v in t.tolist()]
