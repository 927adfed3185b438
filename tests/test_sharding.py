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


def _bench_worker(rank, world, port, q):
    """bench.py's end-of-run reduction with per-rank arms."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys = ["steps", "triggers", "repairs"]
        stats = {"mg": {"steps": 20, "triggers": 3 + rank, "repairs": rank},
                 "bf16": {"steps": 20, "triggers": 0, "repairs": 0}}
        det = {"mg_vs_ao": (64 - rank, 64), "bf16_vs_ao": (rank, 64)}
        tokens = {"mg": 1280, "bf16": 1280 - rank}
        times = {"mg": 100.0 + rank, "bf16": 80.0 - rank, "e2e": 120.0}
        same = sharding.reduce_run(stats, keys, det, tokens, times, probe=[5, 6, 7, 8])
        diff = sharding.reduce_run(stats, keys, det, tokens, times, probe=[5, 6, 7, 8 + rank])
        q.put((rank, same, diff["probe_identical"]))
    finally:
        dist.destroy_process_group()


def test_bench_reduction_two_gloo_ranks():
    """The bench's aggregation path as 2 gloo ranks: stats, determinism counts
    and tokens SUM exactly, device times MAX, and the cross-rank determinism
    probe (the same protected request decoded on every rank) is identical only
    when every rank's sequence is."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = {}
    for _ in ps:
        r, same, ident_diff = q.get(timeout=120)
        out[r] = (same, ident_diff)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        same, ident_diff = out[r]
        assert same["stats"]["mg"] == {"steps": 40, "triggers": 7, "repairs": 1}
        assert same["stats"]["bf16"] == {"steps": 40, "triggers": 0, "repairs": 0}
        assert same["det"] == {"bf16_vs_ao": (1, 128), "mg_vs_ao": (127, 128)}
        assert same["tokens"] == {"bf16": 2559, "mg": 2560}
        assert same["times"] == {"bf16": 80.0, "e2e": 120.0, "mg": 101.0}
        assert same["probe_identical"] is True and ident_diff is False


def test_digest_and_single_rank_probe():
    assert sharding.digest([1, 2, 3]) == sharding.digest([1, 2, 3]) != sharding.digest([1, 2, 4])
    assert 0 <= sharding.digest(range(100)) < 2 ** 62
    assert sharding.all_equal([1, 2]) is True
    r = sharding.reduce_run({"a": {"k": 1}}, ["k"], {"d": (1, 2)}, {"a": 3}, {"a": 1.5}, probe=[1])
    assert r == {"stats": {"a": {"k": 1}}, "det": {"d": (1, 2)}, "tokens": {"a": 3}, "times": {"a": 1.5},
                 "probe_identical": True}
