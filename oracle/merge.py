"""Oracle integer side of model merging: signatures, groups, byte accounting.

Test infrastructure only (see oracle/__init__.py).

* Architectural equivalence (§3.1 "Commonality of layers"):
  two layers can be shared iff they have the same type and identical values for
  the type's defining properties; weights, position and input H x W are not
  part of it.  Only layers with weights (conv, linear, BN) are counted, which
  is how the paper counts "41/73 layers (20 conv, 1 FC, 20 BN)".
* Groups (§4.2 "Merging Heuristic"): every appearance of a layer
  across the workload, with the models it appears in "(and where)" and the total
  memory it consumes; sorted in descending order of that total ("a 100 MB layer
  that appears in 4 models would be earlier than a 120 MB layer that appears 3
  times").  Tie-break (reading R5): per-appearance bytes desc, then
  first appearance (model, position) asc.
* Memory saved by a merge configuration: one copy of each
  shared layer is kept, so a group of n appearances saves (n-1) x its bytes.
* Weights of a merged group come from one member ("initial weights
  ... from a random model that includes that layer"); here an explicit source
  index (default member 0, reading R6).
"""
from __future__ import annotations

from collections import defaultdict

PARAM_OPS = ("conv", "linear", "bn")


def signature(layer):
    """Hashable architectural signature of a layer, or None for param-less ops.

    A conv tied to another layer's parameters (``tie``: Faster R-CNN's RPN head run
    on every FPN level) is that layer applied again, not a layer of its own: None."""
    if "tie" in layer:
        return None
    op = layer["op"]
    if op == "conv":
        return ("conv", layer["cin"], layer["cout"], tuple(layer["k"]), tuple(layer["s"]),
                tuple(layer["p"]), tuple(layer["d"]), layer["groups"], bool(layer["bias"]))
    if op == "linear":
        return ("linear", layer["fin"], layer["fout"], bool(layer["bias"]))
    if op == "bn":
        return ("bn", layer["c"], float(layer["eps"]), float(layer["momentum"]),
                bool(layer["affine"]), bool(layer["track"]))
    return None


def param_count(layer):
    """Number of parameter elements held by a layer (BN: gamma, beta, mean, var)."""
    if "tie" in layer:
        return 0
    op = layer["op"]
    if op == "conv":
        kh, kw = layer["k"]
        return layer["cout"] * (layer["cin"] // layer["groups"]) * kh * kw + (layer["cout"] if layer["bias"] else 0)
    if op == "linear":
        return layer["fout"] * layer["fin"] + (layer["fout"] if layer["bias"] else 0)
    if op == "bn":
        return 4 * layer["c"]
    return 0


def param_bytes(layer, dtype_bytes=2):
    """Exact parameter bytes of a layer in the registered dtype (bf16 = 2 B)."""
    return param_count(layer) * dtype_bytes


def find_shareable(models, dtype_bytes=2):
    """All-appearance signature classes with >= 2 appearances, memory-sorted.

    models: list of layer lists (model id = list index).
    Returns list of dicts: sig, apps [(model, pos)...] (ascending), per_bytes,
    total_bytes = per*n, reclaimable = per*(n-1).
    """
    classes = defaultdict(list)
    for m, layers in enumerate(models):
        for pos, l in enumerate(layers):
            s = signature(l)
            if s is not None:
                classes[s].append((m, pos))
    groups = []
    for s, apps in classes.items():
        if len(apps) < 2:
            continue
        apps = sorted(apps)
        per = param_bytes(models[apps[0][0]][apps[0][1]], dtype_bytes)
        groups.append({"sig": s, "apps": apps, "per_bytes": per,
                       "total_bytes": per * len(apps), "reclaimable": per * (len(apps) - 1)})
    groups.sort(key=lambda g: (-g["total_bytes"], -g["per_bytes"], g["apps"][0]))
    return groups


def bytes_saved(models, merge_groups, dtype_bytes=2):
    """sum over merge groups of (n-1) * bytes of the group's layer."""
    total = 0
    for g in merge_groups:
        m, pos = g["members"][0]
        total += (len(g["members"]) - 1) * param_bytes(models[m][pos], dtype_bytes)
    return total


def validate_merge(models, merge_groups, already=()):
    """Raise ValueError unless every group is a valid merge (same signature,
    n >= 2, no member in two groups, valid ids, param layer)."""
    seen = set(already)
    for gi, g in enumerate(merge_groups):
        mem = g["members"]
        if len(mem) < 2:
            raise ValueError(f"group {gi}: fewer than 2 members")
        src = g.get("source", 0)
        if not 0 <= src < len(mem):
            raise ValueError(f"group {gi}: bad source index")
        sig0 = None
        for (m, pos) in mem:
            if not (0 <= m < len(models) and 0 <= pos < len(models[m])):
                raise ValueError(f"group {gi}: bad member ({m},{pos})")
            s = signature(models[m][pos])
            if s is None:
                raise ValueError(f"group {gi}: member ({m},{pos}) has no weights")
            if sig0 is None:
                sig0 = s
            elif s != sig0:
                raise ValueError(f"group {gi}: signature mismatch at ({m},{pos})")
            if (m, pos) in seen:
                raise ValueError(f"group {gi}: member ({m},{pos}) already merged")
            seen.add((m, pos))
    return seen


def merged_params(models, params, merge_groups):
    """Per-model params after merging: each member holds the source member's weights.

    This is the plain definition of merged execution: one weight copy used by
    every member, i.e. unmerged execution with copied weights.
    """
    out = [[dict(p) for p in ps] for ps in params]
    for g in merge_groups:
        mem = g["members"]
        sm, sp = mem[g.get("source", 0)]
        for (m, pos) in mem:
            out[m][pos] = dict(params[sm][sp])
    return out


def full_merge(groups):
    """The "Optimal" configuration (Fig. upper_memory):
    share every architecturally identical layer, i.e. every group in full."""
    return [{"members": list(g["apps"]), "source": 0} for g in groups]


def cross_model_groups(groups):
    """Cross-model merge groups, the benchmark configuration (R3, SURVEY.md
    §8(a) a3 "full cross-model config"): at most one appearance per model in a group.
    Within a signature class (find_shareable), the k-th appearance in layer order of
    every model that has >= k+1 appearances forms group k, so identical architectures
    pair layer by layer ("which models the layer appears in (and
    where)"); a class of per-model counts c_i saves bytes * (sum c_i - max c_i).
    Weights from the first member (PAPER.md:378 / R6).  Single-member groups are
    dropped (nothing to share)."""
    out = []
    for g in groups:
        by_model = defaultdict(list)
        for (m, pos) in sorted(g["apps"]):
            by_model[m].append((m, pos))
        k = 0
        while True:
            members = [by_model[m][k] for m in sorted(by_model) if len(by_model[m]) > k]
            if len(members) < 2:
                break
            out.append({"members": members, "source": 0})
            k += 1
    return out


def overlap(layers_a, layers_b):
    """Number of architecturally identical layers between two models (multiset
    intersection of signatures), the quantity of Fig. models_overlap."""
    ca, cb = defaultdict(int), defaultdict(int)
    for l in layers_a:
        s = signature(l)
        if s is not None:
            ca[s] += 1
    for l in layers_b:
        s = signature(l)
        if s is not None:
            cb[s] += 1
    return sum(min(ca[s], cb[s]) for s in ca)


def overlap_by_type(layers_a, layers_b):
    ca, cb = defaultdict(int), defaultdict(int)
    for l in layers_a:
        s = signature(l)
        if s is not None:
            ca[s] += 1
    for l in layers_b:
        s = signature(l)
        if s is not None:
            cb[s] += 1
    out = defaultdict(int)
    for s in ca:
        out[s[0]] += min(ca[s], cb[s])
    return dict(out)


def halve(apps):
    """One halving of a group ("halves the current group, eliminating half
    of the layer appearances"): the first ceil(n/2) appearances in (model, position)
    order stay (reading R21: deterministic; a halved group of one appearance cannot
    be shared)."""
    return list(apps[:(len(apps) + 1) // 2])


def incremental_merge(models, retrain, dtype_bytes=2):
    """GEMEL's incremental merging heuristic (§4.2), step by step.

    groups = find_shareable(models) in descending order of total memory.  A
    running configuration starts empty.  Group i is tried with ALL its appearances
    ("attempts to share it across all of the models in which it appears"):
    retrain(running + [candidate]) -> True when every merged model meets its accuracy
    target within the time budget (the pluggable retraining oracle; no training here).
      * success: the candidate joins the running configuration; next group;
      * failure: the group is halved; if the halved appearances (>= 2) consume
        more memory than the next group in the sorted list they are tried next,
        otherwise the group is dropped and the next group is tried.
    Weights of a merged group come from its first member (reading R6).

    Returns (config, log): config = accepted merge groups in acceptance order; log =
    one entry per retraining attempt {"group": index in the sorted list, "members":
    tried appearances, "bytes": their total, "ok": bool}."""
    groups = find_shareable(models, dtype_bytes)
    config, log = [], []
    i = 0
    cur = list(groups[0]["apps"]) if groups else []
    while i < len(groups):
        cand = {"members": [tuple(a) for a in cur], "source": 0}
        ok = bool(retrain(config + [cand]))
        log.append({"group": i, "members": cand["members"], "bytes": groups[i]["per_bytes"] * len(cur), "ok": ok})
        if ok:
            config.append(cand)
            i += 1
            cur = list(groups[i]["apps"]) if i < len(groups) else []
            continue
        half = halve(cur)
        nxt = groups[i + 1]["total_bytes"] if i + 1 < len(groups) else 0
        if len(half) >= 2 and groups[i]["per_bytes"] * len(half) > nxt:
            cur = half
        else:
            i += 1
            cur = list(groups[i]["apps"]) if i < len(groups) else []
    return config, log
