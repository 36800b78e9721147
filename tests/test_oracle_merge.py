"""Pins for oracle/merge.py: paper-printed overlap counts, the cfg1 worked example,
the P:374 ordering example, brute force on tiny random models, and the
closed-form byte accounting."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import merge, model
from workloads import synth, zoo

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _jsonable(sig):
    return json.loads(json.dumps(sig))


@pytest.mark.parametrize("pin", _load("paper_pins.json")["overlap"], ids=lambda p: f"{p['a']}-{p['b']}")
def test_paper_overlap_pins(pin):
    a, b = zoo.build(pin["a"]), zoo.build(pin["b"])
    assert merge.overlap(a, b) == pin["total"]
    assert merge.overlap_by_type(a, b) == pin["by_type"]


def test_vgg16_heavy_hitter_392mb():
    pins = _load("paper_pins.json")
    fc6 = [l for l in zoo.build("vgg16") if l["op"] == "linear"][0]
    assert round(merge.param_bytes(fc6, 4) / 2 ** 20, 2) == pins["vgg16_fc6_fp32_mib"]
    assert merge.param_bytes(fc6, 4) == (25088 * 4096 + 4096) * 4


def test_cfg1_worked_example():
    g = _load("cfg1_find_shareable.json")
    models = [zoo.build("tiny_a"), zoo.build("tiny_b")]
    groups = merge.find_shareable(models)
    assert len(groups) == len(g["groups"])
    for got, exp in zip(groups, g["groups"]):
        assert _jsonable(got["sig"]) == exp["sig"]
        assert [list(a) for a in got["apps"]] == exp["apps"]
        for k in ("per_bytes", "total_bytes", "reclaimable"):
            assert got[k] == exp[k]
    cfgm = merge.full_merge(groups)
    assert merge.bytes_saved(models, cfgm) == g["bytes_saved_bf16"]
    assert merge.bytes_saved(models, cfgm, 4) == g["bytes_saved_fp32"]


def _lin(fin, fout):
    return {"op": "linear", "in": [-1], "fin": fin, "fout": fout, "bias": False}


def test_p374_ordering_example():
    """'a 100 MB layer that appears in 4 models would be earlier than a 120 MB
    layer that appears 3 times', scaled to 100/120 kB."""
    x, y = _lin(100, 500), _lin(120, 500)     # 100,000 B and 120,000 B in bf16
    models = [[dict(x)], [dict(x), dict(y)], [dict(x), dict(y)], [dict(x), dict(y)]]
    groups = merge.find_shareable(models)
    assert [g["per_bytes"] for g in groups] == [100_000, 120_000]
    assert [len(g["apps"]) for g in groups] == [4, 3]


def _random_model(rng, n):
    layers = []
    for i in range(n):
        kind = rng.integers(0, 4)
        src = [i - 1] if i > 0 else [-1]
        if kind == 0:
            k = int(rng.choice([1, 3]))
            layers.append({"op": "conv", "in": src, "cin": int(rng.choice([8, 16])), "cout": int(rng.choice([8, 16])),
                           "k": (k, k), "s": (int(rng.choice([1, 2])),) * 2, "p": (k // 2, k // 2), "d": (1, 1),
                           "groups": 1, "bias": bool(rng.integers(0, 2))})
        elif kind == 1:
            layers.append({"op": "bn", "in": src, "c": int(rng.choice([8, 16])), "eps": 1e-5, "momentum": 0.1,
                           "affine": True, "track": True})
        elif kind == 2:
            layers.append({"op": "linear", "in": src, "fin": int(rng.choice([4, 8])), "fout": int(rng.choice([4, 8])),
                           "bias": bool(rng.integers(0, 2))})
        else:
            layers.append({"op": "relu", "in": src})
    return layers


def _same_arch_bruteforce(a, b):
    """Pairwise architectural equality by direct field comparison (no signature)."""
    if a["op"] != b["op"] or a["op"] not in merge.PARAM_OPS:
        return False
    keys = set(a) | set(b)
    return all(a.get(k) == b.get(k) for k in keys if k != "in")


@pytest.mark.parametrize("seed", range(20))
def test_find_shareable_bruteforce(seed):
    rng = np.random.default_rng(seed)
    models = [_random_model(rng, int(rng.integers(3, 9))) for _ in range(int(rng.integers(2, 5)))]
    apps = [(m, p) for m, ls in enumerate(models) for p in range(len(ls))]
    # equivalence classes from all pairs (union-find)
    parent = {a: a for a in apps}

    def find(a):
        while parent[a] != a:
            a = parent[a]
        return a
    for a, b in itertools.combinations(apps, 2):
        if _same_arch_bruteforce(models[a[0]][a[1]], models[b[0]][b[1]]):
            parent[find(a)] = find(b)
    classes = {}
    for a in apps:
        if models[a[0]][a[1]]["op"] in merge.PARAM_OPS:
            classes.setdefault(find(a), []).append(a)
    expected = sorted(sorted(c) for c in classes.values() if len(c) >= 2)
    got = merge.find_shareable(models)
    assert sorted(g["apps"] for g in got) == expected
    # equivalence relation: every member pair in a group is equal, no cross-group pair is
    for g in got:
        for a, b in itertools.combinations(g["apps"], 2):
            assert _same_arch_bruteforce(models[a[0]][a[1]], models[b[0]][b[1]])
    # sort order: total desc, per desc, first app asc
    keys = [(-g["total_bytes"], -g["per_bytes"], g["apps"][0]) for g in got]
    assert keys == sorted(keys)
    # closed form: full merge saves (all param bytes) - (bytes of one copy per distinct signature)
    allb = sum(merge.param_bytes(l) for ls in models for l in ls)
    uniq = {}
    for ls in models:
        for l in ls:
            s = merge.signature(l)
            if s is not None:
                uniq[s] = merge.param_bytes(l)
    assert merge.bytes_saved(models, merge.full_merge(got)) == allb - sum(uniq.values())


def test_signature_position_independent():
    a = zoo.build("resnet18")
    # the same conv at different positions / different producers has the same signature
    l1, l2 = dict(a[4]), dict(a[7])
    assert l1["op"] == l2["op"] == "conv"
    l2["in"] = [123]
    assert merge.signature(l1) == merge.signature(l2)


def test_validate_merge_rejects():
    models = [zoo.build("tiny_a"), zoo.build("tiny_b")]
    with pytest.raises(ValueError):
        merge.validate_merge(models, [{"members": [(0, 0)]}])
    with pytest.raises(ValueError):
        merge.validate_merge(models, [{"members": [(0, 0), (1, 2)]}])          # signature mismatch
    with pytest.raises(ValueError):
        merge.validate_merge(models, [{"members": [(0, 4), (1, 4)]}])          # 32->32 vs 32->64
    with pytest.raises(ValueError):
        merge.validate_merge(models, [{"members": [(0, 1), (1, 1)]}])          # relu has no weights
    with pytest.raises(ValueError):
        merge.validate_merge(models, [{"members": [(0, 0), (1, 0)]}, {"members": [(0, 0), (1, 0)]}])
    merge.validate_merge(models, [{"members": [(0, 0), (1, 0)]}, {"members": [(0, 2), (1, 2)]}])


def test_merged_equals_unmerged_with_copied_weights():
    models = [zoo.build("tiny_a"), zoo.build("tiny_b")]
    params = [synth.params(m, 1, q) for q, m in enumerate(models)]
    cfgm = merge.full_merge(merge.find_shareable(models))
    mp = merge.merged_params(models, params, cfgm)
    fr = synth.frames(1, 1, 2, 32, 32)
    # unmerged model B with conv0/conv1 weights copied by hand from model A
    pb = [dict(p) for p in params[1]]
    pb[0] = {k: v.copy() for k, v in params[0][0].items()}
    pb[2] = {k: v.copy() for k, v in params[0][2].items()}
    a = model.run(models[1], mp[1], fr)[-1]
    b = model.run(models[1], pb, fr)[-1]
    np.testing.assert_array_equal(a, b)
    # model A (the source) is unchanged by merging
    np.testing.assert_array_equal(model.run(models[0], mp[0], fr)[-1], model.run(models[0], params[0], fr)[-1])


def test_batch_invariance():
    layers = zoo.build("tiny_a")
    p = synth.params(layers, 1, 0)
    fr = synth.frames(1, 0, 3, 32, 32)
    full = model.run(layers, p, fr)[-1]
    for i in range(3):
        one = model.run(layers, p, fr[i:i + 1])[-1]
        np.testing.assert_allclose(one[0], full[i], rtol=1e-13, atol=1e-13)


def test_cfg2_full_merge_savings():
    """Optimal (all identical layers) savings for cfg2 are a large fraction (P:248 range 17.9-86.4%)."""
    models = [zoo.build(n) for n in ("resnet18", "resnet34", "resnet50")]
    groups = merge.find_shareable(models)
    saved = merge.bytes_saved(models, merge.full_merge(groups))
    total = sum(merge.param_bytes(l) for m in models for l in m)
    assert 0.179 <= saved / total <= 0.864
