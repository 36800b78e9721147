"""Seeded synthetic inputs: frames and random-init weights.

Shared by the oracle and the CUDA path (the only module both may use).  It holds
none of the method's arithmetic -- only random-number draws and the storage
rounding that *defines* the inputs (weights are bf16 values by construction).

Recipe:
  * frames: uint8 RGB HWC, uniform 0..255, Philox keyed by (cfg, stream).
  * conv / linear weight: Kaiming-normal on fan-in, gain sqrt(2) when followed
    by ReLU, sqrt(2/(1+0.1^2)) by LeakyReLU(0.1), 1 otherwise; rounded to bf16
    (RNE) once, so both sides consume identical values.
  * bias: U(-0.05, 0.05), bf16-rounded.
  * Detector head convs / linears (feeding a YOLO, SSD, RPN or Fast R-CNN box decode) use gain 0.1: a random darknet trunk grows
    activations to std ~10 by its last stage, and trained heads emit t = O(1);
    gain 1 would overflow exp(t) in the decode.
  * BN: gamma U(0.5,1.5), beta N(0,0.1), mean N(0,0.1), var U(0.5,1.5), fp32.
    A BN that ends a residual branch (first operand of an ``add``, directly or
    through its activation) draws gamma from U(0.1,0.3) instead, so 36-block ResNets keep O(1) activations (random
    weights are not trained; the paper uses trained weights).
"""
from __future__ import annotations

import numpy as np


def round_bf16(x):
    """Round float32 values to the nearest bf16 (ties to even); returns float32."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(a.shape)


def _rng(*key):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([int(k) & 0xFFFFFFFF for k in key])))


def frames(cfg_seed, stream, n, h, w):
    """uint8 [n, h, w, 3] frames for one camera stream."""
    g = _rng(1000 * cfg_seed + stream, 7)
    return g.integers(0, 256, size=(n, h, w, 3), dtype=np.uint8)


def _gain_after(layers, i):
    """Kaiming gain from the activation that consumes layer i (skipping BN)."""
    consumers = [j for j, l in enumerate(layers) if i in l["in"]]
    if consumers and all(layers[j]["op"] in ("yolo", "ssd_decode", "rpn_level", "box_post") for j in consumers):
        return 0.1                   # detector head: keeps t = O(1) over a random trunk (no exp overflow)
    for j in consumers:
        op = layers[j]["op"]
        if op == "bn":
            return _gain_after(layers, j)
        if op == "relu":
            return np.sqrt(2.0)
        if op == "leaky":
            return np.sqrt(2.0 / (1.0 + layers[j]["slope"] ** 2))
    return 1.0


def params(layers, *key):
    """Per-layer parameter dicts (float32 numpy arrays) for a layer list.

    conv  : {"w": [cout, cin/groups, kh, kw], "b": [cout] (if bias)}
    linear: {"w": [fout, fin], "b": [fout] (if bias)}
    bn    : {"gamma","beta","mean","var": [c]}
    others, and convs tied to another layer's parameters: {}
    """
    out = []
    for i, l in enumerate(layers):
        g = _rng(*key, i)
        op = l["op"]
        if "tie" in l:
            out.append({})               # applies layer l["tie"]'s parameters (zoo: tie)
        elif op == "conv":
            kh, kw = l["k"]
            fan_in = (l["cin"] // l["groups"]) * kh * kw
            std = _gain_after(layers, i) / np.sqrt(fan_in)
            w = g.standard_normal((l["cout"], l["cin"] // l["groups"], kh, kw)) * std
            p = {"w": round_bf16(w)}
            if l["bias"]:
                p["b"] = round_bf16(g.uniform(-0.05, 0.05, l["cout"]))
            out.append(p)
        elif op == "linear":
            std = _gain_after(layers, i) / np.sqrt(l["fin"])
            w = g.standard_normal((l["fout"], l["fin"])) * std
            p = {"w": round_bf16(w)}
            if l["bias"]:
                p["b"] = round_bf16(g.uniform(-0.05, 0.05, l["fout"]))
            out.append(p)
        elif op == "bn":
            c = l["c"]
            # a BN that ends a residual branch, directly (ResNet) or through its
            # activation (darknet shortcut: conv-BN-leaky, then add)
            acts = [j for j, m in enumerate(layers) if m["op"] in ("relu", "leaky") and m["in"] == [i]]
            ends_branch = any(m["op"] == "add" and (m["in"][0] == i or m["in"][0] in acts) for m in layers)
            lo, hi = (0.1, 0.3) if ends_branch else (0.5, 1.5)
            out.append({"gamma": g.uniform(lo, hi, c).astype(np.float32),
                        "beta": (g.standard_normal(c) * 0.1).astype(np.float32),
                        "mean": (g.standard_normal(c) * 0.1).astype(np.float32),
                        "var": g.uniform(0.5, 1.5, c).astype(np.float32)})
        elif op == "l2norm":
            out.append({"scale": np.full(l["c"], 20.0, np.float32)})   # torchvision's init
        else:
            out.append({})
    return out
