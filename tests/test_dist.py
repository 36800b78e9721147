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
    res = [q.get(timeout=10) for _ in range(5)]
    assert all(ok for _, ok in res), res
    assert sorted(k for k, _ in res) == ["bcast", "bcast", "gather", "seed", "seed"]
