"""C ABI on the CPU: the library loads, exports every symbol include/gemel.h
declares, and its host-side integer work (signatures, groups, sort, bytes
saved, schema/merge validation) is bit-exact against the oracle."""
import os
import re

import numpy as np
import pytest

from oracle import merge as om
from workloads import synth, zoo

G = pytest.importorskip("paper_2201_07705_b200.gemel")

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "gemel.h")


def test_exports_every_declared_symbol():
    src = open(HDR).read()
    declared = set(re.findall(r"\b(gemel_[a-z_]+)\s*\(", src))
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(G._lib, name), name
    assert declared == set(G.EXPORTED)


def _ctx_with(models, stream_ids=None, res=(32, 32)):
    ctx = G.gemel_create()
    for i, layers in enumerate(models):
        params = synth.params(layers, 0, i)
        sid = i if stream_ids is None else stream_ids[i]
        assert G.gemel_register_model(ctx, layers, params, sid, *res) == i
    return ctx


def _norm_oracle(groups):
    return [(g["per_bytes"], g["total_bytes"], g["reclaimable"], [tuple(a) for a in g["apps"]]) for g in groups]


def _norm_lib(groups):
    return [(g["per_bytes"], g["total_bytes"], g["reclaimable"], [tuple(a) for a in g["apps"]]) for g in groups]


@pytest.mark.parametrize("names,res", [(("tiny_a", "tiny_b"), (32, 32)),
                                       (("resnet18", "resnet34", "resnet50"), (224, 224)),
                                       (("vgg16", "vgg19", "vgg16", "vgg19", "vgg16", "vgg19"), (224, 224)),
                                       (("vgg16", "alexnet"), (224, 224)),
                                       (("resnet101", "resnet152", "resnet50"), (64, 64))])
def test_find_shareable_and_bytes_saved_bit_exact(names, res):
    models = [zoo.build(n) for n in names]
    ctx = _ctx_with(models, res=res)
    try:
        got = G.gemel_find_shareable(ctx)
        exp = om.find_shareable(models)
        assert _norm_lib(got) == _norm_oracle(exp)
        cfg = om.full_merge(exp)
        saved = G.gemel_apply_merge(ctx, [{"members": g["members"], "source": 0} for g in cfg])
        assert saved == om.bytes_saved(models, cfg)
        st = G.gemel_stats(ctx)
        assert st["bytes_saved"] == saved
        assert st["registered_bytes"] == sum(om.param_bytes(l) for m in models for l in m)
        assert st["n_merged_layers"] == sum(len(g["members"]) - 1 for g in cfg)
    finally:
        G.gemel_destroy(ctx)


def test_cfg1_worked_example_through_abi():
    import json
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg1_find_shareable.json")))
    ctx = _ctx_with([zoo.build("tiny_a"), zoo.build("tiny_b")])
    try:
        got = G.gemel_find_shareable(ctx)
        assert [[list(a) for a in g["apps"]] for g in got] == [g["apps"] for g in gold["groups"]]
        assert [g["per_bytes"] for g in got] == [g["per_bytes"] for g in gold["groups"]]
        assert G.gemel_apply_merge(ctx, [{"members": g["apps"]} for g in got]) == gold["bytes_saved_bf16"]
    finally:
        G.gemel_destroy(ctx)


@pytest.mark.parametrize("seed", range(10))
def test_random_models_match_oracle(seed):
    from tests.test_oracle_merge import _random_model  # noqa: F401 (same generator as the oracle pin)
    rng = np.random.default_rng(100 + seed)
    # the C ABI validates shapes, so chain layers with consistent channel counts
    models = []
    for _ in range(int(rng.integers(2, 5))):
        layers, c = [], 3
        for i in range(int(rng.integers(2, 7))):
            src = [i - 1] if i else [-1]
            kind = int(rng.integers(0, 3))
            if kind == 0:
                co = int(rng.choice([8, 16]))
                k = int(rng.choice([1, 3]))
                layers.append({"op": "conv", "in": src, "cin": c, "cout": co, "k": (k, k), "s": (1, 1),
                               "p": (k // 2, k // 2), "d": (1, 1), "groups": 1, "bias": bool(rng.integers(0, 2))})
                c = co
            elif kind == 1:
                layers.append({"op": "bn", "in": src, "c": c, "eps": 1e-5, "momentum": 0.1, "affine": True,
                               "track": True})
            else:
                layers.append({"op": "relu", "in": src})
        models.append(layers)
    ctx = _ctx_with(models, res=(8, 8))
    try:
        assert _norm_lib(G.gemel_find_shareable(ctx)) == _norm_oracle(om.find_shareable(models))
    finally:
        G.gemel_destroy(ctx)


def test_apply_merge_validation_all_or_nothing():
    ctx = _ctx_with([zoo.build("tiny_a"), zoo.build("tiny_b")])
    try:
        good = {"members": [(0, 0), (1, 0)]}
        bad_sig = {"members": [(0, 4), (1, 4)]}
        with pytest.raises(G.GemelError) as e:
            G.gemel_apply_merge(ctx, [good, bad_sig])
        assert e.value.code == G.E_MERGE and "signature" in str(e.value)
        assert G.gemel_stats(ctx)["n_merged_layers"] == 0          # nothing applied
        for bad in ([{"members": [(0, 0)]}], [{"members": [(0, 1), (1, 1)]}], [{"members": [(0, 0), (5, 0)]}],
                    [{"members": [(0, 0), (1, 0)], "source": 2}], [good, good]):
            with pytest.raises(G.GemelError) as e:
                G.gemel_apply_merge(ctx, bad)
            assert e.value.code == G.E_MERGE
        assert G.gemel_apply_merge(ctx, [good]) == 896
        with pytest.raises(G.GemelError):                            # already merged
            G.gemel_apply_merge(ctx, [good])
        assert G.gemel_apply_merge(ctx, [{"members": [(0, 2), (1, 2)], "source": 1}]) == 9280
        assert G.gemel_stats(ctx)["bytes_saved"] == 10176
    finally:
        G.gemel_destroy(ctx)


def test_register_schema_errors_name_position():
    ctx = G.gemel_create()
    try:
        layers = zoo.build("tiny_a")
        params = synth.params(layers, 0, 0)
        bad = [dict(l) for l in layers]
        bad[2] = dict(bad[2], cin=17)                     # conv cin mismatch at op 2
        with pytest.raises(G.GemelError) as e:
            G.gemel_register_model(ctx, bad, params, 0, 32, 32)
        assert e.value.code == G.E_SCHEMA and "op 2" in str(e.value)
        bad = [dict(l) for l in layers]
        bad[7] = dict(bad[7], fin=100)                   # linear in_features mismatch
        with pytest.raises(G.GemelError) as e:
            G.gemel_register_model(ctx, bad, params, 0, 32, 32)
        assert "op 7" in str(e.value)
        bad = [dict(l) for l in layers]
        bad[3] = dict(bad[3], **{"in": [5]})              # not topological
        with pytest.raises(G.GemelError) as e:
            G.gemel_register_model(ctx, bad, params, 0, 32, 32)
        assert e.value.code == G.E_SCHEMA
        assert G.gemel_stats(ctx)["n_models"] == 0
    finally:
        G.gemel_destroy(ctx)


def test_plan_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    ctx = _ctx_with([zoo.build("tiny_a"), zoo.build("tiny_b")])
    try:
        with pytest.raises(G.GemelError) as e:
            G.gemel_plan(ctx, [2, 2])
        assert e.value.code == G.E_CUDA
    finally:
        G.gemel_destroy(ctx)


def test_frcnn_registration_groups_and_ties():
    """Faster R-CNN through the ABI (tied RPN head, detector-stage ops): registered
    bytes = the oracle's 41,861,526 elements x 2 B, find_shareable / full-merge bytes
    bit-exact against the oracle (tied convs are not layers), a tied conv cannot be a
    merge member, and bad ties / detector-stage wiring fail with the op position."""
    models = [zoo.build("frcnn_r50_fpn"), zoo.build("frcnn_r50_fpn"), zoo.build("yolov3")]
    ctx = _ctx_with(models, res=(128, 128))
    try:
        st = G.gemel_stats(ctx)
        assert st["n_param_layers"] == 121 + 121 + 147
        assert st["registered_bytes"] == sum(om.param_bytes(l) for m in models for l in m)
        got = G.gemel_find_shareable(ctx)
        exp = om.find_shareable(models)
        assert _norm_lib(got) == _norm_oracle(exp)
        cfg = om.full_merge(exp)
        assert G.gemel_apply_merge(ctx, [{"members": g["members"], "source": 0} for g in cfg]) == \
            om.bytes_saved(models, cfg)
        tied = next(i for i, l in enumerate(models[0]) if "tie" in l)
        with pytest.raises(G.GemelError) as e:
            G.gemel_apply_merge(ctx, [{"members": [(0, tied), (1, tied)]}])
        assert e.value.code == G.E_MERGE
    finally:
        G.gemel_destroy(ctx)
    layers = zoo.build("frcnn_r50_fpn")
    params = synth.params(layers, 0, 0)
    tied = next(i for i, l in enumerate(layers) if "tie" in l)
    cases = [
        (tied, dict(layers[tied], tie=tied + 1)),                            # tie to a later op
        (tied, dict(layers[tied], tie=next(i for i, l in enumerate(layers) if l["op"] == "bn"))),   # not a conv
        (tied, dict(layers[tied], cout=128, tie=layers[tied]["tie"])),       # hyperparameters differ
    ]
    pos_roi = next(i for i, l in enumerate(layers) if l["op"] == "roi_align")
    cases.append((pos_roi, dict(layers[pos_roi], **{"in": [layers[pos_roi]["in"][1]] + layers[pos_roi]["in"][1:]})))
    pos_bp = next(i for i, l in enumerate(layers) if l["op"] == "box_post")
    cases.append((pos_bp, dict(layers[pos_bp], classes=90)))                 # logits width != classes
    for pos, bad_layer in cases:
        bad = [dict(l) for l in layers]
        bad[pos] = bad_layer
        ctx = G.gemel_create()
        try:
            with pytest.raises(G.GemelError) as e:
                G.gemel_register_model(ctx, bad, params, 0, 128, 128)
            assert e.value.code in (G.E_SCHEMA, G.E_UNSUPPORTED) and f"op {pos}" in str(e.value), (pos, str(e.value))
        finally:
            G.gemel_destroy(ctx)
