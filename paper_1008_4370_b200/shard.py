"""Frame sharding across GPUs: one process per GPU, frames are independent.

Two partitions of the frames:

* ``strong`` (default): a FIXED global batch of F frames (BASELINE.json configs[3], [4]: "frames
  sharded over 1/2/4/8 GPUs") is split into contiguous ranges aligned to the 256-frame noise
  chunks of ``synth`` -- rank g of G takes [g*F/G, (g+1)*F/G) rounded to chunk boundaries, so every
  rank draws whole chunks and a frame's LLRs do not depend on G;
* ``weak``: every rank decodes its own F frames, global indices [g*F, (g+1)*F).

There is no collective in the decoding loop.  After decoding, ONE all-reduce sums the counter vector
``COUNTERS`` (frames, converged, frame / symbol / bit errors against the sent codeword, undetected
errors, frame-iterations, numerical events, ...) and one takes the maximum of the per-rank device
times.  ``gather_rows`` is an optional (untimed) all-gather of per-frame outputs for parity checks.
"""
from __future__ import annotations

CHUNK = 256  # synth.CHUNK: the noise of frame f is drawn from Philox keyed by (seed, f // 256)

# counters summed over ranks; every one is an integer count
COUNTERS = ("frames", "ok", "frame_iters", "frame_err", "sym_err", "bit_err", "undetected", "events",
            "launches", "e2e_frame_iters")


def frame_range(rank: int, world: int, frames: int, scaling: str = "weak", chunk: int = CHUNK) -> tuple[int, int]:
    """Global frame indices [first, last) of ``rank``.

    scaling="weak": ``frames`` per rank, [rank*frames, (rank+1)*frames).
    scaling="strong": ``frames`` is the global batch; contiguous chunk-aligned ranges that cover
    [0, frames) exactly (the last rank takes the remainder; ranks may be empty when frames < world*chunk).
    """
    if not (0 <= rank < world) or frames < 1:
        raise ValueError("bad rank / world / frames")
    if scaling == "weak":
        return rank * frames, (rank + 1) * frames
    if scaling != "strong":
        raise ValueError("scaling must be 'weak' or 'strong'")
    nchunks = -(-frames // chunk)

    def start(g):
        return min(frames, (g * nchunks // world) * chunk)

    return start(rank), (frames if rank == world - 1 else start(rank + 1))


def error_counts(hard, ok, sent=None, events=None) -> dict:
    """Counts of one decoded batch against the sent codeword (all-zero when ``sent`` is None):
    frame errors (estimate != sent, PAPER.md:141-144 defines success as "forms a codeword", so a
    converged frame on a wrong codeword is an *undetected* error and still a frame error), symbol
    errors, bit errors (popcount of hard XOR sent), undetected errors, converged frames, events.
    Torch tensors on any device; returns python ints."""
    import torch

    h = hard.to(torch.int32)
    if sent is not None:
        h = h ^ sent.to(device=hard.device, dtype=torch.int32)
    wrong = h != 0
    ferr = wrong.any(dim=1)
    pop = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64, device=hard.device)
    okb = ok.to(torch.bool)
    return {"frames": int(hard.shape[0]), "ok": int(okb.sum().item()), "frame_err": int(ferr.sum().item()),
            "sym_err": int(wrong.sum().item()), "bit_err": int(pop[h.long()].sum().item()),
            "undetected": int((ferr & okb).sum().item()),
            "events": 0 if events is None else int(events.to(torch.int64).sum().item())}


def reduce_stats(counters: dict, times: dict, dist=None, device=None) -> tuple[dict, dict]:
    """Sum ``counters`` and take the max of ``times`` over ranks (identity without a process group).
    Counters travel in one int64 tensor, times in one float64 tensor (one all-reduce each)."""
    import torch

    ck, tk = sorted(counters), sorted(times)
    c = torch.tensor([int(counters[k]) for k in ck], dtype=torch.int64, device=device)
    t = torch.tensor([float(times[k]) for k in tk], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return ({k: int(v) for k, v in zip(ck, c.tolist())}, {k: v for k, v in zip(tk, t.tolist())})


def gather_rows(t, dist=None, frames_per_rank=None):
    """All-gather a per-frame tensor [F_r, ...] from every rank in rank order (ranks may hold
    different F_r: ``frames_per_rank`` lists them; rows are padded to the largest for the collective).
    Identity without a process group."""
    import torch

    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return t
    world = dist.get_world_size()
    sizes = frames_per_rank or [t.shape[0]] * world
    mx = max(sizes)
    pad = torch.zeros((mx, *t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:n] for p, n in zip(parts, sizes)])
