"""Multi-GPU host logic on CPU: request sharding and the
end-of-run SUM / MAX collectives, run as 2 gloo ranks over 127.0.0.1."""
import os
import socket

import pytest

from paper_2605_30218_b200 import inputs, sharding


def test_rank_requests_partition():
    for world in (1, 2, 4, 8):
        for per in (1, 3, 64):
            seen = []
            for r in range(world):
                ids = list(sharding.rank_requests(r, world, per))
                assert len(ids) == per
                assert all(sharding.request_rank(i, per) == r for i in ids)
                seen += ids
            assert sorted(seen) == list(range(world * per))      # every request exactly once
    with pytest.raises(ValueError):
        sharding.rank_requests(2, 2, 4)


def test_rank_prompts_are_the_global_requests():
    # rank r's prompt j is global request r*B + j (seed 7 + request id)
    B, L, V = 3, 5, 1000
    glob = inputs.prompts(2 * B, L, V, seed=7)
    for r in range(2):
        loc = inputs.prompts(B, L, V, seed=7 + sharding.rank_requests(r, 2, B)[0])
        assert loc == glob[r * B:(r + 1) * B]


def test_aggregate_single_rank_is_identity():
    c, t = sharding.aggregate([1, 2, 3], [0.5, 2.0])
    assert c == [1, 2, 3] and t == [0.5, 2.0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # per-rank stats: counters differ by rank, times too
        counters = [10 * (rank + 1), rank, 7, 2 ** 40 + rank]
        times = [1.0 + rank, 5.0 - rank]
        q.put((rank, sharding.aggregate(counters, times)))
    finally:
        dist.destroy_process_group()


def test_aggregate_two_gloo_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        c, t = out[r]
        assert c == [30, 1, 14, 2 ** 41 + 1]      # SUM, exact in int64
        assert t == [2.0, 5.0]                     # MAX over ranks
