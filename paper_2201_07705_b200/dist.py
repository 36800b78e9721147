"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL).

The merged workload partitions by camera stream: each rank
runs its own queries on its own streams with no per-step activation exchange
(merging never shares intermediates).  Either every rank runs a
copy of the configuration on its own streams (weak scaling), or one
configuration's queries are split across the ranks by `partition_queries`
(strong scaling, e.g. the 32-stream cfg5 over 8 GPUs).  Two collectives remain:
  * setup: the merged weight arena is broadcast from rank 0 once, so every GPU
    holds the single merged copy (north_star: "placed once per GPU with an
    NCCL broadcast over NVLink");
  * per step: each rank's result slab (logits of its streams) is gathered to
    rank 0.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def stream_seed(stream_id: int, rank: int) -> int:
    """Frame-generator stream key of a rank's stream (disjoint across ranks)."""
    return stream_id + 1000 * rank


def broadcast_weights(arena: torch.Tensor, src: int = 0) -> None:
    """Place the merged weights once per GPU: rank `src`'s arena -> every rank."""
    dist.broadcast(arena, src=src)


def partition_queries(costs, arch, world, slack=0.05):
    """Greedy bin packing of queries onto `world` GPUs.

    costs[q]: algorithmic cost of query q (FLOPs per step); arch[q]: its
    architecture.  Queries are placed largest first, each on the rank with the
    least load after placement -- among ranks within `slack` of that least load,
    one that already hosts the same architecture is preferred, so sharers are
    co-located and their merged layers union their batches (place
    models that share layers together).  Deterministic (ties by index).
    Returns the sorted query indices of every rank."""
    order = sorted(range(len(costs)), key=lambda q: (-costs[q], q))
    load = [0.0] * world
    members = [[] for _ in range(world)]
    for q in order:
        best = min(load[r] + costs[q] for r in range(world))
        cands = [r for r in range(world) if load[r] + costs[q] <= best * (1.0 + slack)]
        same = [r for r in cands if any(arch[p] == arch[q] for p in members[r])]
        r = min(same or cands, key=lambda r: (load[r], r))
        members[r].append(q)
        load[r] += costs[q]
    return [sorted(m) for m in members]


class ResultGather:
    """Per-step gather of every rank's result slab to rank `dst` on a dedicated comm
    stream, so the collective of step k overlaps step k+1's compute (SURVEY.md
    §8(e)).  The slab is packed on the compute stream after the step, the comm stream
    waits for it; the next pack waits for the previous gather (the slab is reused).
    Slabs are padded to `max_numel` (the largest over ranks) when ranks hold
    different queries."""

    def __init__(self, outs: dict, rank: int, world: int, dst: int = 0, max_numel: int = 0, compute_stream=None):
        self.keys = sorted(outs)
        self.rank, self.world, self.dst = rank, world, dst
        self.n = sum(outs[k].numel() for k in self.keys)
        dev = outs[self.keys[0]].device
        self.slab = torch.zeros(max(self.n, max_numel), dtype=torch.float32, device=dev)
        self.recv = [torch.empty_like(self.slab) for _ in range(world)] if rank == dst else None
        self.cuda = dev.type == "cuda"
        self.sent = None
        if self.cuda:
            self.compute = compute_stream if compute_stream is not None else torch.cuda.current_stream(dev)
            self.comm = torch.cuda.Stream(device=dev)
            self.packed = torch.cuda.Event()

    def __call__(self, outs: dict):
        if not self.cuda:                                  # CPU tensors (gloo): synchronous
            torch.cat([outs[k].reshape(-1) for k in self.keys], out=self.slab[:self.n])
            dist.gather(self.slab, self.recv, dst=self.dst)
            return self.recv
        with torch.cuda.stream(self.compute):
            if self.sent is not None:
                self.compute.wait_event(self.sent)        # the previous gather has read the slab
            torch.cat([outs[k].reshape(-1) for k in self.keys], out=self.slab[:self.n])
            self.packed.record(self.compute)
        self.comm.wait_event(self.packed)
        with torch.cuda.stream(self.comm):
            dist.gather(self.slab, self.recv, dst=self.dst)
            self.sent = torch.cuda.Event()
            self.sent.record(self.comm)
        return self.recv

    def wait(self):
        """Block the compute stream until the last gather completed."""
        if self.cuda and self.sent is not None:
            self.compute.wait_event(self.sent)
