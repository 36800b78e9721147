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
            sigs = {om.signature(models[m][pos]) for m, pos in mem}
            assert len(sigs) == 1, f"union {mem} joins different architectures"
            sources = {src.get(x, x) for x in mem}
            assert len(sources) == 1, f"union {mem} joins layers that do not share one weight copy"
    return True
