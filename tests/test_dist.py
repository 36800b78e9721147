"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host logic used by
bench.py: weight broadcast from rank 0 and the per-step result gather."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2201_07705_b200.dist import ResultGather, broadcast_weights, stream_seed
    try:
        arena = torch.full((1000,), float(rank + 1), dtype=torch.uint8)
        broadcast_weights(arena, src=0)
        ok_bcast = bool((arena == 1).all())
        outs = {0: torch.full((2, 3), 10.0 * rank), 1: torch.full((2, 5), 10.0 * rank + 1)}
        g = ResultGather(outs, rank, world)
        recv = g(outs)
        if rank == 0:
            got = [r.tolist() for r in recv]
            exp = [[10.0 * r] * 6 + [10.0 * r + 1] * 10 for r in range(world)]
            q.put(("gather", got == exp))
        # --shard: ranks hold different queries, slabs padded to the largest
        outs = {0: torch.full((2, 3 + rank), 5.0 + rank)}
        g = ResultGather(outs, rank, world, max_numel=2 * (3 + world - 1))
        recv = g(outs)
        if rank == 0:
            got = [r.tolist() for r in recv]
            exp = [[5.0 + r] * (2 * (3 + r)) + [0.0] * (2 * (world - 1 - r)) for r in range(world)]
            q.put(("gather_padded", got == exp))
        q.put(("bcast", ok_bcast))
        q.put(("seed", stream_seed(2, rank) != stream_seed(2, 1 - rank)))
    finally:
        dist.destroy_process_group()


def test_broadcast_and_gather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = [q.get(timeout=10) for _ in range(6)]
    assert all(ok for _, ok in res), res
    assert sorted(k for k, _ in res) == ["bcast", "bcast", "gather", "gather_padded", "seed", "seed"]


def test_partition_queries_cfg5():
    """--shard bin packing of the 32-stream cfg5 over 2-8 GPUs: every
    query exactly once, deterministic, load within the greedy bound (max load <= mean +
    largest query), and sharers co-located when balance allows (two equal halves of one
    architecture over 2 ranks stay together)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2201_07705_b200.dist import partition_queries
    from workloads import configs
    cfg = configs.CONFIGS[5]
    costs = bench.query_costs(cfg)
    arch = [n for n, _ in cfg["queries"]]
    for world in (2, 4, 8):
        part = partition_queries(costs, arch, world)
        assert sorted(q for r in part for q in r) == list(range(len(costs)))
        assert part == partition_queries(costs, arch, world)
        loads = [sum(costs[q] for q in r) for r in part]
        assert max(loads) <= sum(costs) / world + max(costs)
    part = partition_queries([4.0, 4.0, 1.0, 1.0, 1.0, 1.0], ["a", "a", "b", "b", "b", "b"], 2)
    assert all(len({["a", "a", "b", "b", "b", "b"][q] for q in r if q < 2}) <= 1 for r in part)
    part = partition_queries([1.0, 1.0, 1.0, 1.0], ["x", "y", "x", "y"], 2)
    assert sorted(map(tuple, part)) == [(0, 2), (1, 3)]           # same architecture co-located
