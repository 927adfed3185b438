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

import hashlib


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


def digest(seq) -> int:
    """62-bit digest of a token sequence (cross-rank identity checks)."""
    h = hashlib.blake2b(b",".join(str(int(t)).encode() for t in seq), digest_size=8).digest()
    return int.from_bytes(h, "little") >> 2


def all_equal(values, device=None) -> bool:
    """True when every rank passed the same list of ints (MAX and -MIN agree):
    one MAX all-reduce over (v, -v); trivially true on one rank."""
    import torch
    import torch.distributed as dist

    values = [int(v) for v in values]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return True
    v = torch.tensor(values + [-x for x in values], dtype=torch.int64, device=device)
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    n = len(values)
    return all(int(v[i]) == -int(v[n + i]) for i in range(n))


def reduce_run(stats: dict, keys, det: dict, tokens: dict, times: dict, probe=None, device=None) -> dict:
    """The end-of-run reduction of bench.py: per-arm MarginGate
    counters (stats[arm][key]), determinism counts det[name] = (equal,
    protected), committed tokens per arm -- all SUMmed; per-arm device times
    MAXed; probe = the token sequence of the request every rank decodes
    (cross-rank determinism: the same protected request on every rank must be
    bit-identical, whatever shares its batch).  Arms and names are reduced in
    sorted order, so every rank packs the same layout."""
    arms, dn, tn = sorted(stats), sorted(det), sorted(times)
    vec = [int(stats[a][k]) for a in arms for k in keys]
    vec += [int(x) for n in dn for x in det[n]]
    vec += [int(tokens[a]) for a in arms]
    c, t = aggregate(vec, [times[n] for n in tn], device=device)
    out = {"stats": {}, "det": {}, "tokens": {}, "times": dict(zip(tn, t))}
    i = 0
    for a in arms:
        out["stats"][a] = dict(zip(keys, c[i:i + len(keys)]))
        i += len(keys)
    for n in dn:
        out["det"][n] = (c[i], c[i + 1])
        i += 2
    for a in arms:
        out["tokens"][a] = c[i]
        i += 1
    out["probe_identical"] = None if probe is None else all_equal([digest(probe)], device=device)
    return out
