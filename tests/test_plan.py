"""Host-side planner (dry plan, no GPU) validated by the oracle's plan checker:
every layer runs once, topological order, unions only over one shared weight."""
import pytest

from oracle import merge as om
from oracle import plan as oplan
from workloads import synth, zoo

G = pytest.importorskip("paper_2201_07705_b200.gemel")


def _zero_params(layers):
    """Shapes-only params (the planner never reads values)."""
    import numpy as np
    out = []
    for l in layers:
        if l["op"] == "conv":
            p = {"w": np.zeros((l["cout"], l["cin"], *l["k"]), np.float32)}
            if l["bias"]:
                p["b"] = np.zeros(l["cout"], np.float32)
        elif l["op"] == "linear":
            p = {"w": np.zeros((l["fout"], l["fin"]), np.float32)}
            if l["bias"]:
                p["b"] = np.zeros(l["fout"], np.float32)
        elif l["op"] == "bn":
            p = {k: np.ones(l["c"], np.float32) for k in ("gamma", "beta", "mean", "var")}
        elif l["op"] == "l2norm":
            p = {"scale": np.ones(l["c"], np.float32)}
        else:
            p = {}
        out.append(p)
    return out


def _plan(names, res, batch, merge="full"):
    models = [zoo.build(n) for n in names]
    ctx = G.gemel_create(flags=G.FLAG_DRY_PLAN)
    for i, m in enumerate(models):
        G.gemel_register_model(ctx, m, _zero_params(m), i, res, res)
    groups = G.gemel_find_shareable(ctx)
    cfg = [{"members": g["apps"], "source": 0} for g in groups] if merge == "full" else []
    if cfg:
        G.gemel_apply_merge(ctx, cfg)
    info = G.gemel_plan(ctx, [batch] * len(models))
    dump = G.gemel_plan_dump(ctx)
    G.gemel_destroy(ctx)
    return models, cfg, info, dump


@pytest.mark.parametrize("names,res", [(("tiny_a", "tiny_b"), 32),
                                       (("resnet18", "resnet34", "resnet50"), 224),
                                       (("vgg16", "vgg19", "vgg16", "vgg19"), 224),
                                       (("resnet50", "resnet101", "resnet152"), 64),
                                       (("yolov3", "yolov3", "tiny_yolov3"), 416),
                                       (("ssd300", "ssd300"), 300),
                                       (("frcnn_r50_fpn", "frcnn_r50_fpn", "yolov3"), 128)])
@pytest.mark.parametrize("merge", ["full", "none"])
def test_plan_valid(names, res, merge):
    models, cfg, info, dump = _plan(names, res, 2, merge)
    assert oplan.validate(models, cfg, dump)
    if merge == "none":
        assert info["n_union_problems"] == 0
    else:
        assert info["n_union_problems"] > 0
    assert info["unmerged_weight_bytes"] == sum(om.param_bytes(l) for m in models for l in m)
    assert info["unmerged_weight_bytes"] - info["unique_weight_bytes"] == om.bytes_saved(models, cfg)


def test_cfg1_stems_run_once_over_both_streams():
    models, cfg, info, dump = _plan(("tiny_a", "tiny_b"), 32, 2)
    unions = [p for L in dump["launches"] if L["kind"] == "gemm" for p in L["problems"] if len(p["members"]) > 1]
    assert sorted(sorted(map(tuple, p["members"])) for p in unions) == [[(0, 0), (1, 0)], [(0, 2), (1, 2)]]
    assert all(p["M"] == 2 * 2 * 32 * 32 or p["M"] == 2 * 2 * 16 * 16 for p in unions)


def test_validator_catches_violations():
    models, cfg, info, dump = _plan(("tiny_a", "tiny_b"), 32, 2)
    import copy
    bad = copy.deepcopy(dump)
    bad["nodes"][-1]["layers"] = []                       # a layer never runs
    with pytest.raises(AssertionError):
        oplan.validate(models, cfg, bad)
    bad = copy.deepcopy(dump)
    for n in bad["nodes"]:
        n["level"] = 0                                     # breaks topological order
    with pytest.raises(AssertionError):
        oplan.validate(models, cfg, bad)
    with pytest.raises(AssertionError):                    # union without a shared weight
        oplan.validate(models, [], dump)


def _plan_budget(names, res, batch, merge, budget_frac):
    models = [zoo.build(n) for n in names]
    total = sum(om.param_bytes(l) for m in models for l in m)
    budget = int(total * budget_frac)
    ctx = G.gemel_create(flags=G.FLAG_DRY_PLAN, weight_budget_bytes=budget)
    for i, m in enumerate(models):
        G.gemel_register_model(ctx, m, _zero_params(m), i, res, res)
    groups = om.find_shareable(models)   # merge configs come from the oracle, not the library
    cfg = om.cross_model_groups(groups) if merge == "cross" else []
    if cfg:
        G.gemel_apply_merge(ctx, cfg)
    info = G.gemel_plan(ctx, [batch] * len(models))
    dump = G.gemel_plan_dump(ctx)
    G.gemel_destroy(ctx)
    return models, cfg, info, dump, budget


@pytest.mark.parametrize("names,res,frac", [(("vgg16", "vgg19", "vgg16"), 224, 0.5),
                                            (("vgg16", "vgg19", "vgg16"), 224, 0.75),
                                            (("resnet18", "resnet34", "resnet50"), 224, 0.5),
                                            (("resnet18", "resnet34", "resnet50"), 224, 0.3),
                                            (("yolov3", "tiny_yolov3"), 416, 0.5),
                                            (("yolov3", "tiny_yolov3"), 416, 0.3)])
def test_swap_plan_invariants(names, res, frac):
    """Budgeted plans: unmerged weights exceed the budget, so a
    pinned set plus a swap ring streams the rest every step -- validated by the oracle."""
    models, cfg, info, dump, budget = _plan_budget(names, res, 2, "none", frac)
    assert oplan.validate(models, cfg, dump)
    assert oplan.validate_swap(dump, budget)
    assert info["n_swapped"] > 0 and info["swap_bytes_per_step"] > 0
    assert info["weight_arena_bytes"] <= budget
    # minimal swap: everything above the budget is streamed (up to the ring's headroom)
    assert info["swap_bytes_per_step"] >= info["unique_weight_bytes"] - budget


def test_merging_removes_swap():
    """PAPER.md:1068 on B200: with a 50% budget VGG16+VGG19+VGG16 unmerged must stream
    weights every step; cross-model merged it fits and streams nothing."""
    _, _, info_u, _, budget = _plan_budget(("vgg16", "vgg19", "vgg16"), 224, 2, "none", 0.5)
    _, _, info_m, dump_m, _ = _plan_budget(("vgg16", "vgg19", "vgg16"), 224, 2, "cross", 0.5)
    assert info_u["swap_bytes_per_step"] > 0
    assert info_m["swap_bytes_per_step"] == 0 and info_m["n_swapped"] == 0
    assert oplan.validate_swap(dump_m, budget)


def test_budget_below_double_buffered_ring_is_an_error():
    """30% of VGG16+VGG19+VGG16 (252 MB) cannot double-buffer the 205 MB fc6 weight."""
    with pytest.raises(G.GemelError) as e:
        _plan_budget(("vgg16", "vgg19", "vgg16"), 224, 2, "none", 0.3)
    assert e.value.code == G.E_NOMEM
