"""Frame sharding across GPUs: one process per GPU, each
decoding its own contiguous frame range with its own handle.  Frames are
independent, so the data path has no collective; the only exchange is an
end-of-run reduction of a few counters and the max-over-ranks step time.

Host-side plumbing only (torch.distributed); no decoding happens here.
"""
from __future__ import annotations


def frame_range(rank: int, world: int, frames_per_rank: int):
    """Weak scaling: rank r owns global frames [r * F, (r + 1) * F)."""
    if not (0 <= rank < world) or frames_per_rank < 0:
        raise ValueError("bad rank/world/frames")
    return rank * frames_per_rank, (rank + 1) * frames_per_rank


def split_range(rank: int, world: int, total: int):
    """Strong scaling: a contiguous near-equal split of [0, total)."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("bad rank/world/total")
    q, r = divmod(total, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


COUNTERS = ("frames", "frame_errors", "bit_errors", "pops", "switches")


def reduce_counters(counts: dict, device=None) -> dict:
    """Sum int64 counters over ranks (all_reduce SUM); identity without a group."""
    import torch
    import torch.distributed as dist
    vec = torch.tensor([int(counts.get(k, 0)) for k in COUNTERS], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(vec, op=dist.ReduceOp.SUM)
    return {k: int(v) for k, v in zip(COUNTERS, vec.tolist())}


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. the device-timed step), as the contract requires."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
