"""Frame sharding across GPUs: one process per GPU, frames are independent.

Rank r of a world of G decodes the contiguous global frame range
[r*F, (r+1)*F) ("weak" scaling: F frames per rank).  There is no collective in
the decoding loop; after decoding, one all-reduce sums the per-rank counters and
one takes the maximum of the per-rank device times.
"""
from __future__ import annotations

# counters summed over ranks, in this order
COUNTERS = ("frame_iters", "ok", "frames", "launches", "e2e_frame_iters")


def frame_range(rank: int, world: int, frames_per_rank: int) -> tuple[int, int]:
    """Global frame indices [first, last) of ``rank``."""
    if not (0 <= rank < world) or frames_per_rank < 1:
        raise ValueError("bad rank / world / frames_per_rank")
    return rank * frames_per_rank, (rank + 1) * frames_per_rank


def reduce_stats(counters: dict, times: dict, dist=None, device=None) -> tuple[dict, dict]:
    """Sum ``counters`` and take the max of ``times`` over ranks (identity without a process group).
    Values are carried in one float64 tensor per reduction (exact for counts below 2^53)."""
    import torch

    ck, tk = sorted(counters), sorted(times)
    c = torch.tensor([float(counters[k]) for k in ck], dtype=torch.float64, device=device)
    t = torch.tensor([float(times[k]) for k in tk], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return ({k: v for k, v in zip(ck, c.tolist())}, {k: v for k, v in zip(tk, t.tolist())})
