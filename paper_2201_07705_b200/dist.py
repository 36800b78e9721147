"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL).

The merged workload partitions by camera stream: each rank
runs its own queries on its own streams with no per-step activation exchange
(merging never shares intermediates).  Two collectives remain:
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


class ResultGather:
    """Per-step gather of every rank's result slab to rank `dst` (fixed-size slabs)."""

    def __init__(self, outs: dict, rank: int, world: int, dst: int = 0):
        self.keys = sorted(outs)
        self.rank, self.world, self.dst = rank, world, dst
        n = sum(outs[k].numel() for k in self.keys)
        dev = outs[self.keys[0]].device
        self.slab = torch.empty(n, dtype=torch.float32, device=dev)
        self.recv = [torch.empty_like(self.slab) for _ in range(world)] if rank == dst else None

    def __call__(self, outs: dict):
        torch.cat([outs[k].reshape(-1) for k in self.keys], out=self.slab)
        dist.gather(self.slab, self.recv, dst=self.dst)
        return self.recv
