"""Oracle model execution: one model, layer by layer, NumPy fp64.

Test infrastructure only (see oracle/__init__.py).  Each query runs its own
model on its own stream's frames; merging shares weights, never intermediates
(PAPER.md:203), so a merged workload's result is, per query, exactly this
function evaluated with the merged weights (see merge.merged_params).

``emulate_bf16=True`` rounds to bf16 (RNE) every value the B200 path stores in
bf16 ("storage points", reading R7): the preprocessed frame, the end
of every fused chain ``conv|linear -> [bn] -> [add] -> [relu|leaky]`` (darknet:
``conv -> bn -> leaky -> add``), pool outputs.  The final layer's output, a
YOLO head's raw output and its decode stay fp64 (the device stores them fp32).
"""
from __future__ import annotations

import numpy as np

from . import ops


def round_bf16(x):
    """fp64 -> nearest bf16 value (ties to even), returned as fp64.

    Two-step: fp64 -> fp32 (RNE) -> bf16 (RNE on the fp32 bit pattern).  The
    device rounds fp32 accumulators, so this is the same rounding it performs.
    """
    a = np.asarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64).reshape(a.shape)


def consumers(layers):
    cons = [[] for _ in layers]
    for j, l in enumerate(layers):
        for i in l["in"]:
            if i >= 0:
                cons[i].append(j)
    return cons


def storage_points(layers):
    """Boolean per layer: is this layer's output materialised (bf16) on the device?"""
    cons = consumers(layers)
    stored = [True] * len(layers)
    for i, l in enumerate(layers):
        c = cons[i]
        if len(c) != 1:
            continue
        nxt = layers[c[0]]
        op, nop = l["op"], nxt["op"]
        if op in ("conv", "linear"):
            if nop == "bn" or nop in ("relu", "leaky") or (nop == "add" and nxt["in"][0] == i):
                stored[i] = False
        elif op == "bn" and i > 0 and layers[l["in"][0]]["op"] in ("conv", "linear") \
                and not stored[l["in"][0]]:
            if nop in ("relu", "leaky") or (nop == "add" and nxt["in"][0] == i):
                stored[i] = False
        elif op == "add" and nop in ("relu", "leaky"):
            src = l["in"][0]
            if src >= 0 and not stored[src]:
                stored[i] = False
        elif op in ("relu", "leaky") and nop == "add" and nxt["in"][0] == i:
            src = l["in"][0]             # darknet shortcut: conv -> bn -> leaky -> add, one chain
            if src >= 0 and layers[src]["op"] in ("conv", "linear", "bn") and not stored[src]:
                stored[i] = False
        elif op == "flatten":
            stored[i] = False            # a view: no new storage, nothing to round
        elif op == "upsample" and nop in ("concat", "add"):
            stored[i] = False            # read by the concat copy / the residual add directly (exact either way)
    # fp32 storage (never bf16-rounded): a head feeding a decode (YOLO, SSD, RPN, the
    # Fast R-CNN box decode), the decode itself, a concat of decodes (the model's
    # detection output), the top-k rows and the RPN proposals
    decode = ("yolo", "ssd_decode", "rpn_level", "box_post")
    for i, l in enumerate(layers):
        if cons[i] and all(layers[j]["op"] in decode for j in cons[i]):
            stored[i] = False
        if l["op"] in decode + ("topk", "rpn_merge", "det_cand", "det_nms") or (l["op"] == "concat" and all(layers[j]["op"] in decode for j in l["in"])):
            stored[i] = False
    return stored


def run(layers, params, frames_u8, emulate_bf16=False):
    """Evaluate a model; returns the list of every layer's output (fp64, NCHW or [N,F])."""
    x0 = ops.preprocess(frames_u8)
    if emulate_bf16:
        x0 = round_bf16(x0)
    stored = storage_points(layers) if emulate_bf16 else None
    vals = []
    last = len(layers) - 1
    for i, (l, p) in enumerate(zip(layers, params)):
        ins = [x0 if j < 0 else vals[j] for j in l["in"]]
        if "tie" in l:
            p = params[l["tie"]]         # the tied layer's parameters (zoo: tie)
        op = l["op"]
        x = ins[0]
        if op == "conv":
            y = ops.conv2d(x, p["w"], p.get("b"), l["s"], l["p"], l["d"], l["groups"])
        elif op == "bn":
            y = ops.batchnorm(x, p["gamma"], p["beta"], p["mean"], p["var"], l["eps"])
        elif op == "relu":
            y = ops.relu(x)
        elif op == "leaky":
            y = ops.leaky_relu(x, l["slope"])
        elif op == "maxpool":
            y = ops.maxpool2d(x, l["k"], l["s"], l["p"], l["d"], l["ceil"], l.get("darknet", False))
        elif op == "gap":
            y = ops.adaptive_avgpool2d(x, l["out"])
        elif op == "add":
            y = ops.add(ins[0], ins[1])
        elif op == "concat":
            y = ops.concat(ins)
        elif op == "upsample":
            y = ops.upsample_nearest(x, l["scale"])
        elif op == "flatten":
            y = ops.flatten(x)
        elif op == "linear":
            y = ops.linear(x, p["w"], p.get("b"))
        elif op == "yolo":
            y = ops.yolo_decode(x, l["anchors"], l["classes"], x0.shape[2:])
        elif op == "topk":
            y = ops.topk_rows(x, l["k"], l["fields"], l["score"])
        elif op == "det_cand":
            y = ops.det_candidates(x, l["fmt"], l["fields"], l["score_thresh"], l["min_size"])
        elif op == "det_nms":
            y = ops.det_nms(x, l["iou"], l["max_det"])
        elif op == "l2norm":
            y = ops.l2norm(x, p["scale"], l["eps"])
        elif op == "ssd_decode":
            y = ops.ssd_decode(ins[0], ins[1], l["wh"], l["step"], l["classes"], l["weights"], x0.shape[2:])
        elif op == "rpn_level":
            y = ops.rpn_level(ins[0], ins[1], l["size"], l["ratios"], l["pre_n"], l["nms"], l["min_size"],
                              x0.shape[2:])
        elif op == "rpn_merge":
            y = ops.rpn_merge(ins, l["post_n"])
        elif op == "roi_align":
            y = ops.multiscale_roi_align(ins[1:], ins[0], l["out"], l["sampling"], l["canonical"], x0.shape[2:])
        elif op == "box_post":
            y = ops.box_post(ins[0], ins[1], ins[2], l["classes"], l["weights"], x0.shape[2:])
        else:
            raise ValueError(f"unknown op {op}")
        if emulate_bf16 and stored[i] and i != last:
            y = round_bf16(y)
        vals.append(y)
    return vals


def shapes(layers, in_hw, cin=3):
    """Per-layer output shapes (C,H,W) / (F,) for an input of size in_hw (oracle's own)."""
    out = []
    for l in layers:
        ins = [(cin,) + tuple(in_hw) if j < 0 else out[j] for j in l["in"]]
        out.append(ops.out_shape(l, ins))
    return out
