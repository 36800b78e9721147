"""Oracle validator for execution plans dumped by the library (gemel_plan_dump).

Test infrastructure only (see oracle/__init__.py).  A valid step plan for a
merged workload (SURVEY.md §8(c) "plan validator"):

  * every layer of every model runs exactly once per step (flatten is a view);
  * order is topological: a node's inputs are produced at a strictly earlier
    scheduler level (GEMM problems of one launch may depend on each other, the
    kernel waits on completion counters);
  * a batch-union problem only joins layers that are architecturally identical
     and bound to ONE weight copy by the merge configuration
    (PAPER.md:203, 376-378), from distinct models -- models never share
    intermediates, only weights.
"""
from __future__ import annotations

from . import merge as om


def _source_of(merge_cfg):
    src = {}
    for g in merge_cfg:
        s = tuple(g["members"][g.get("source", 0)])
        for m in g["members"]:
            src[tuple(m)] = s
    return src


def validate(models, merge_cfg, dump):
    """Raise AssertionError describing the first violated invariant."""
    covered = {}
    for ni, n in enumerate(dump["nodes"]):
        for pos in n["layers"]:
            key = (n["model"], pos)
            assert key not in covered, f"layer {key} covered by nodes {covered[key]} and {ni}"
            covered[key] = ni
    for m, layers in enumerate(models):
        for pos, l in enumerate(layers):
            if l["op"] == "flatten":
                assert (m, pos) not in covered, f"flatten {(m, pos)} should be a view"
                continue
            assert (m, pos) in covered, f"layer {(m, pos)} ({l['op']}) never runs"

    # position of every node in the launch sequence: (launch index, index within the launch)
    order = {}
    for li, L in enumerate(dump["launches"]):
        if L["kind"] == "gemm":
            for pi, p in enumerate(L["problems"]):
                for m, pos in p["members"]:
                    order[("gemm", m, pos)] = (li, pi)
        else:
            for ni, (m, pos) in enumerate(L["nodes"]):
                order[(L["kind"], m, pos)] = (li, ni)
    node_key = []
    for n in dump["nodes"]:
        first = n["layers"][0] if n["layers"] else None
        if n["kind"] == "preprocess":
            first = n["output"][1] if n["output"][1] < -1 else -1
            first = -2 - first if first < -1 else -1
        k = order.get((n["kind"], n["model"], first))
        assert k is not None, f"node {n['kind']} of model {n['model']} is in no launch"
        node_key.append(k)
    # the node (and launch position) that produces each value (model, pos)
    produced_at = {}
    for ni, n in enumerate(dump["nodes"]):
        if n["output"] is not None:
            produced_at[tuple(n["output"])] = (n["level"], node_key[ni], n["kind"])
    # flatten views resolve to their input
    def resolve(model, pos):
        while pos >= 0 and models[model][pos]["op"] == "flatten":
            pos = models[model][pos]["in"][0]
        return pos
    for ni, n in enumerate(dump["nodes"]):
        for v in n["inputs"]:
            if v is None:
                continue
            key = (v[0], resolve(v[0], v[1]) if v[1] >= 0 else v[1])
            assert key in produced_at, f"node {ni} reads {key}, which no node produces"
            lvl, (pl, pp), pkind = produced_at[key]
            cl, cp = node_key[ni]
            assert lvl < n["level"], f"node {ni} (level {n['level']}) reads {key} produced at level {lvl}"
            # launch order: an earlier launch, or an earlier problem of the same GEMM launch
            assert pl < cl or (pl == cl and pkind == "gemm" and n["kind"] == "gemm" and pp < cp), \
                f"node {ni} at launch {(cl, cp)} reads {key} produced at launch {(pl, pp)}"

    src = _source_of(merge_cfg)
    for L in dump["launches"]:
        if L["kind"] != "gemm":
            continue
        for p in L["problems"]:
            mem = [tuple(x) for x in p["members"]]
            if len(mem) < 2:
                continue
            models_in = [m for m, _ in mem]
            assert len(set(models_in)) == len(models_in), f"union {mem} has two layers of one model"
            # a tied conv (zoo ``tie``) applies its target's weights: judge it as that layer
            mem = [(m, models[m][pos].get("tie", pos)) for m, pos in mem]
            sigs = {om.signature(models[m][pos]) for m, pos in mem}
            assert len(sigs) == 1, f"union {mem} joins different architectures"
            sources = {src.get(x, x) for x in mem}
            assert len(sources) == 1, f"union {mem} joins layers that do not share one weight copy"
    return True


def validate_swap(dump, budget):
    """Weight-residency invariants of a budgeted plan (SPEC's
    residency invariants): the weight arena fits the budget; pinned tensors and
    ring slots do not overlap; every streamed tensor is copied before the first
    launch that reads it, into a slot inside the ring, and a copy never overwrites
    a slot whose previous occupant is still read by a later or concurrent launch."""
    sw = dump["swap"]
    W = sw["weights"]
    if budget:
        assert sw["weight_arena_bytes"] <= budget, (sw["weight_arena_bytes"], budget)
    uses = {}
    for li, L in enumerate(dump["launches"]):
        if L["kind"] != "gemm":
            continue
        for p in L["problems"]:
            uses.setdefault(p["wkey"], []).append(li)
    ring0, ring1 = sw["ring_off"], sw["ring_off"] + sw["ring_bytes"]
    pinned = sorted((w["offset"], w["offset"] + w["bytes"]) for w in W if not w["swapped"])
    for (a0, a1), (b0, _) in zip(pinned, pinned[1:]):
        assert a1 <= b0, "pinned weights overlap"
    for a0, a1 in pinned:
        assert a1 <= ring0 or a0 >= ring1, "pinned weight inside the swap ring"
    streamed = sorted((w for w in W if w["swapped"]), key=lambda w: w["copy_order"])
    assert sum(w["bytes"] for w in streamed) == sw["swap_bytes"]
    for k, w in enumerate(W):
        if not w["swapped"]:
            continue
        lu = uses[k]
        assert w["first_launch"] == min(lu) and w["last_launch"] == max(lu), (k, w, lu)
        assert ring0 <= w["offset"] and w["offset"] + w["bytes"] <= ring1, f"weight {k} outside the ring"
        assert w["wait_launch"] < w["first_launch"], f"weight {k} copied after its first use"
    for j, a in enumerate(streamed):
        for b in streamed[j + 1:]:
            if a["offset"] < b["offset"] + b["bytes"] and b["offset"] < a["offset"] + a["bytes"]:
                assert b["wait_launch"] >= a["last_launch"], "a copy overwrites a slot still being read"
                assert b["first_launch"] > a["last_launch"]
    return True


def min_swap_bytes(sizes, avail, align=256):
    """Minimal weight bytes streamed per step under an HBM budget, by exhaustive
    search (reading R14): choose the resident
    (pinned) subset P of the weight tensors; the rest stream every step through a
    ring that double-buffers the largest streamed tensor, so P is feasible iff
    sum(P) + 2 * max(streamed) <= avail (sizes rounded up to `align`).  Returns the
    minimum over feasible P of the streamed bytes (unrounded), or None if no P is
    feasible.  Exponential: for instances of a few tensors only."""
    n = len(sizes)
    al = [(s + align - 1) // align * align for s in sizes]
    best = None
    for mask in range(1 << n):
        pinned = sum(al[i] for i in range(n) if mask >> i & 1)
        streamed = [i for i in range(n) if not mask >> i & 1]
        ring = 2 * max((al[i] for i in streamed), default=0)
        if pinned + ring <= avail:
            b = sum(sizes[i] for i in streamed)
            best = b if best is None else min(best, b)
    return best


def lcs_length(a, b, match):
    """Longest common subsequence of sequences a, b under the predicate match(x, y),
    exact dynamic programming (the number of layers two chains can union)."""
    n, m = len(a), len(b)
    T = [[0] * (m + 1) for _ in range(n + 1)]
    for i in range(n):
        for j in range(m):
            T[i + 1][j + 1] = T[i][j] + 1 if match(a[i], b[j]) else max(T[i][j + 1], T[i + 1][j])
    return T[n][m]


def scs_length(a, b, match):
    """Shortest common supersequence length = |a| + |b| - LCS: the number of distinct
    GEMM problems when two chains union every layer pair bound to one weight
    (SURVEY.md §8(a) a5 / §8(c)(iii) "waves = SCS length by exact DP for 2 chains")."""
    return len(a) + len(b) - lcs_length(a, b, match)
