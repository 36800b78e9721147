"""Merged multi-model workload on one GPU: the public Python API over the C ABI.

PyTorch is used only for device memory (the two arenas), pinned host staging
and streams; every step of the path runs in libgemel's kernels.
"""
from __future__ import annotations

import torch

from . import gemel as G


def full_merge_config(groups):
    """Share every architecturally identical layer (the paper's "Optimal"
    configuration, PAPER.md:445 / Fig. upper_memory): each group in
    full, weights from its first appearance (reading R6)."""
    return [{"members": list(g["apps"]), "source": 0} for g in groups]


def cross_model_merge_config(groups):
    """Cross-model groups (at most one appearance per model), SURVEY.md §8(c-ii)'s
    benchmark reading (R3): within a find_shareable signature class, the
    k-th appearance of every model that has one forms group k -- order-preserving,
    so identical architectures pair layer by layer.  Source = member 0."""
    cfg = []
    for g in groups:
        per_model = {}
        for m, pos in sorted(tuple(a) for a in g["apps"]):
            per_model.setdefault(m, []).append((m, pos))
        depth = max(len(v) for v in per_model.values())
        for k in range(depth):
            members = [v[k] for _, v in sorted(per_model.items()) if len(v) > k]
            if len(members) >= 2:
                cfg.append({"members": members, "source": 0})
    return cfg


class MergedWorkload:
    """Register queries, merge, plan and bind one GPU's share of a workload.

    queries: list of (layers, params, stream_id); res: (h, w), or {stream: (h, w)}
    when streams differ (every model of a stream sees its frames); batch: frames per
    stream per step (int or {stream: n}); merge: "full" (every group in full),
    "cross" (cross-model groups, cross_model_merge_config), "none" or an explicit
    list of merge groups ({"members": [(model, pos), ...], "source": i});
    weight_budget: HBM bytes for weights (0 = all resident); above it a pinned set
    stays resident and the rest stream every step (a10) from pinned host memory
    (weight_source "host") or from a peer GPU's HBM over NVLink (weight_source "peer",
    source_device).
    """

    def __init__(self, queries, res, batch, merge="full", device=None, weight_budget=0, weight_source="host",
                 source_device=None):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.stream = torch.cuda.Stream(device=self.device)
        src = G.SOURCE_PEER if weight_source == "peer" else G.SOURCE_HOST
        self.ctx = G.gemel_create(self.device.index, self.stream.cuda_stream, weight_budget_bytes=int(weight_budget),
                                  weight_source=src,
                                  source_device=self.device.index if source_device is None else source_device)
        self.res = res
        self.models = []
        for layers, params, sid in queries:
            h, w = res[sid] if isinstance(res, dict) else res
            self.models.append((G.gemel_register_model(self.ctx, layers, params, sid, h, w), sid, layers))
        self.groups = G.gemel_find_shareable(self.ctx)
        if merge == "full":
            cfg = full_merge_config(self.groups)
        elif merge == "cross":
            cfg = cross_model_merge_config(self.groups)
        elif merge == "none":
            cfg = []
        else:
            cfg = merge
        self.merge_config = cfg
        self.bytes_saved = G.gemel_apply_merge(self.ctx, cfg) if cfg else 0
        streams = sorted({sid for _, sid, _ in self.models})
        nstream = max(streams) + 1
        if isinstance(batch, int):
            batch = {s: batch for s in streams}
        self.batch = batch
        self.plan = G.gemel_plan(self.ctx, [batch.get(s, 0) for s in range(nstream)])
        self.w_arena = torch.empty(max(self.plan["weight_arena_bytes"], 256), dtype=torch.uint8, device=self.device)
        self.a_arena = torch.empty(max(self.plan["act_arena_bytes"], 256), dtype=torch.uint8, device=self.device)
        G.gemel_bind_arenas(self.ctx, self.w_arena.data_ptr(), self.w_arena.numel(),
                            self.a_arena.data_ptr(), self.a_arena.numel())
        # per-frame output features (logits / decoded boxes) from the library's own shape inference
        self.out_features = {}
        for mid, _, layers in self.models:
            d = G.gemel_value_desc(self.ctx, mid, len(layers) - 1)
            self.out_features[mid] = d["h"] * d["w"] * d["c"]
        self.streams = streams

    # ------------------------------------------------------------------ results
    def alloc_outputs(self, on_host=False):
        outs = {}
        for mid, sid, _ in self.models:
            shape = (self.batch[sid], self.out_features[mid])
            if on_host:
                outs[mid] = torch.empty(shape, dtype=torch.float32, pin_memory=True)
            else:
                outs[mid] = torch.empty(shape, dtype=torch.float32, device=self.device)
        return outs

    def infer(self, frames, outs, on_host=False):
        """frames: {stream: uint8 tensor [B, H, W, 3]} (device, or pinned host if
        on_host); outs: {model: fp32 tensor [B, F]} from alloc_outputs.  Async on
        self.stream."""
        ins = [(s, frames[s].data_ptr(), frames[s].shape[0], on_host) for s in self.streams]
        res = [(m, t.data_ptr(), t.numel() * 4, on_host) for m, t in outs.items()]
        G.gemel_infer(self.ctx, ins, res)

    def read_value(self, model_id, op_pos):
        return G.gemel_read_value(self.ctx, model_id, op_pos)

    def launch_list(self):
        return G.gemel_launch_list(self.ctx)

    def set_profiling(self, on):
        G.gemel_set_profiling(self.ctx, on)

    def weight_view(self):
        return G.gemel_weight_view(self.ctx)

    def close(self):
        if self.ctx:
            G.gemel_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
