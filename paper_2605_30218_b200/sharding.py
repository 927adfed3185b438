"""Request sharding and the end-of-run statistics collective.

Requests are independent units: global request i runs on rank i // B (B rows
per GPU), every rank holds a full weight replica and its own caches, so the
decode path has no data-path collective.  The only collectives are at the end
of a run: one SUM over the int64 counters (MarginGate stats, determinism
counts) and one MAX over the per-arm device times (whole-job throughput =
all ranks' tokens / the slowest rank's time).  torch.distributed carries them
(NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations


def rank_requests(rank: int, world: int, per_rank: int) -> range:
    """Global request ids decoded by `rank` (request i -> rank i // per_rank)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return range(rank * per_rank, (rank + 1) * per_rank)


def request_rank(request: int, per_rank: int) -> int:
    return request // per_rank


def aggregate(counters, times, device=None):
    """SUM the int64 counters and MAX the float times over the default process
    group; identity when torch.distributed is not initialised (one rank)."""
    import torch
    import torch.distributed as dist

    counters = [int(v) for v in counters]
    times = [float(t) for t in times]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return counters, times
    cv = torch.tensor(counters, dtype=torch.int64, device=device)
    dist.all_reduce(cv, op=dist.ReduceOp.SUM)
    tv = torch.tensor(times, dtype=torch.float64, device=device)
    dist.all_reduce(tv, op=dist.ReduceOp.MAX)
    return cv.tolist(), tv.tolist()
