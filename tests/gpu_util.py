"""Shared helpers for the GPU parity tests (tests only)."""
from __future__ import annotations

import numpy as np

from oracle import merge as om
from oracle import model as omodel
from oracle import ops
from workloads import synth, zoo

TOL = 2e-2       # north_star: max |gpu - oracle| / (|oracle| + 1e-3) <= 2e-2
FLOOR = 1e-3


def rel_err(gpu, ref):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    if gpu.size == 0:
        return 0.0
    return float(np.max(np.abs(gpu - ref) / (np.abs(ref) + FLOOR)))


def normwise_err(gpu, ref):
    """max |gpu - ref| / max |ref| (the floor scaled to the output's magnitude)."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    return float(np.abs(gpu - ref).max() / max(np.abs(ref).max(), FLOOR))


def to_nchw(v):
    """GPU value [n, h, w, c] (float32) -> oracle NCHW layout (fp64)."""
    return np.ascontiguousarray(v.transpose(0, 3, 1, 2)).astype(np.float64)


def like(g, ref):
    """Device value in NCHW reshaped to the oracle's shape ([n, f] vectors)."""
    return g.reshape(ref.shape) if ref.ndim == 2 else g


def make_queries(cfg, names, seed_cfg=None):
    seed = cfg if seed_cfg is None else seed_cfg
    models = [zoo.build(n) for n in names]
    params = [synth.params(m, seed, q) for q, m in enumerate(models)]
    return models, params


def oracle_layer(l, p, ins):
    op = l["op"]
    x = ins[0]
    if op == "conv":
        return ops.conv2d(x, p["w"], p.get("b"), l["s"], l["p"], l["d"], l["groups"])
    if op == "bn":
        return ops.batchnorm(x, p["gamma"], p["beta"], p["mean"], p["var"], l["eps"])
    if op == "relu":
        return ops.relu(x)
    if op == "leaky":
        return ops.leaky_relu(x, l["slope"])
    if op == "maxpool":
        return ops.maxpool2d(x, l["k"], l["s"], l["p"], l["d"], l["ceil"], l.get("darknet", False))
    if op == "gap":
        return ops.adaptive_avgpool2d(x, l["out"])
    if op == "add":
        return ops.add(ins[0], ins[1])
    if op == "flatten":
        return ops.flatten(x)
    if op == "linear":
        return ops.linear(x, p["w"], p.get("b"))
    raise ValueError(op)


def teacher_forced(read_value, mid, layers, params, frames_u8):
    """Compare every value the device stores with the oracle's layer applied to
    the device's own (bf16) inputs.  Returns {pos: rel_err}."""
    stored = omodel.storage_points(layers)
    last = len(layers) - 1
    errs = {}
    g_in = to_nchw(read_value(mid, -1))
    errs[-1] = rel_err(g_in, ops.preprocess(frames_u8))
    vals = {-1: g_in}
    for i, l in enumerate(layers):
        y = oracle_layer(l, params[i], [vals[j] for j in l["in"]])
        if stored[i] or i == last:
            g = like(to_nchw(read_value(mid, i)), y)
            errs[i] = rel_err(g, y)
            vals[i] = g
        else:
            vals[i] = y
    return errs


def oracle_outputs(models, params, merge_cfg, frames_by_model, emulate_bf16=False):
    mp = om.merged_params(models, params, merge_cfg) if merge_cfg else params
    return [omodel.run(m, p, f, emulate_bf16=emulate_bf16)[-1] for m, p, f in zip(models, mp, frames_by_model)]
