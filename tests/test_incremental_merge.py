"""N3: the incremental merging planner (§4.2).

The oracle (oracle.merge.incremental_merge) is pinned by closed forms and a
hand-worked example written from the paper's text; the library's native planner
(gemel_incremental_merge, driving gemel_apply_merge) must reproduce the oracle's
attempt log and accepted configuration exactly (integer work: bit-exact) for any
deterministic retraining oracle.  No training happens: the retraining step is a
pluggable callback."""
import zlib

import pytest

from oracle import merge as om
from workloads import configs, zoo

G = pytest.importorskip("paper_2201_07705_b200.gemel")
from tests.test_plan import _zero_params  # noqa: E402


def test_always_success_is_the_full_merge():
    models = [zoo.build(n) for n in ("resnet18", "resnet34", "resnet50")]
    cfg, log = om.incremental_merge(models, lambda c: True)
    groups = om.find_shareable(models)
    assert [g["members"] for g in cfg] == [list(g["apps"]) for g in groups]
    assert len(log) == len(groups) and all(e["ok"] for e in log)
    assert om.bytes_saved(models, cfg) == om.bytes_saved(models, om.full_merge(groups))


def test_always_failure_attempt_count_closed_form():
    """Nothing is accepted; group i is tried at n, ceil(n/2), ceil(n/4), ... appearances
    while the halved appearances are >= 2 and outweigh group i+1's total."""
    models = [zoo.build(n) for n in ("vgg16", "vgg19", "vgg16", "vgg11")]
    cfg, log = om.incremental_merge(models, lambda c: False)
    assert cfg == []
    groups = om.find_shareable(models)
    expect = 0
    for i, g in enumerate(groups):
        n = len(g["apps"])
        nxt = groups[i + 1]["total_bytes"] if i + 1 < len(groups) else 0
        expect += 1
        while (n + 1) // 2 >= 2 and g["per_bytes"] * ((n + 1) // 2) > nxt:
            n = (n + 1) // 2
            expect += 1
    assert len(log) == expect


def test_paper_example_exact_log():
    """The P:374 example with exact byte sizes: X = 100 KiB per appearance in 4 models,
    Y = 120 KiB per appearance in 3 models, Z = 90 KiB in 2 models.  Sorted: X (400),
    Y (360), Z (180).  Oracle rejects any candidate with 4 members and accepts the rest:
      X x4 fail -> half = 2 appearances (200) <= Y's 360 -> drop X;
      Y x3 ok;  Z x2 ok:  three attempts, bytes saved = 2*120 + 1*90 KiB.
    (Linear layers here are never executed: only signatures and bytes matter.)"""
    K = 1024
    # linear fin -> fout with bf16 bytes 2 * fin * fout
    x = {"op": "linear", "fin": 100, "fout": 512, "bias": False}     # 102 400 B
    y = {"op": "linear", "fin": 120, "fout": 512, "bias": False}     # 122 880 B
    z = {"op": "linear", "fin": 90, "fout": 512, "bias": False}      # 92 160 B

    def model(parts):
        layers = []
        for p in parts:
            d = dict(p)
            d["in"] = [-1]
            layers.append(d)
        return layers
    models = [model([x, y, z]), model([x, y, z]), model([x, y]), model([x])]
    groups = om.find_shareable(models)
    assert [(len(g["apps"]), g["per_bytes"]) for g in groups] == [(4, 100 * K), (3, 120 * K), (2, 90 * K)]
    cfg, log = om.incremental_merge(models, lambda c: len(c[-1]["members"]) < 4)
    assert [(e["group"], len(e["members"]), e["ok"]) for e in log] == [(0, 4, False), (1, 3, True), (2, 2, True)]
    assert om.bytes_saved(models, cfg) == 2 * 120 * K + 90 * K
    # rejecting 3+ members: X is dropped as before; a failing Y is halved to 2 appearances
    # (240 > Z's 180) and retried, then Z
    cfg, log = om.incremental_merge(models, lambda c: len(c[-1]["members"]) < 3)
    assert [(e["group"], len(e["members"]), e["ok"]) for e in log] == [
        (0, 4, False), (1, 3, False), (1, 2, True), (2, 2, True)]
    assert om.bytes_saved(models, cfg) == 120 * K + 90 * K


def _crc_oracle(cfg):
    """Deterministic pseudo-random retraining outcome of the candidate (last entry)."""
    return zlib.crc32(repr(cfg[-1]["members"]).encode()) % 3 != 0


@pytest.mark.parametrize("cfg_id", [2, 3, 4])
@pytest.mark.parametrize("oracle_fn", ["crc", "budget"])
def test_library_matches_oracle(cfg_id, oracle_fn):
    cfg = configs.CONFIGS[cfg_id]
    models = [zoo.build(n) for n, _ in cfg["queries"]]
    if oracle_fn == "crc":
        retrain = _crc_oracle
    else:   # accuracy "degrades" with the number of shared appearances in the running config
        def retrain(c):
            return sum(len(g["members"]) for g in c) <= 60 and len(c[-1]["members"]) <= 4
    ref_cfg, ref_log = om.incremental_merge(models, retrain)
    ctx = G.gemel_create(flags=G.FLAG_DRY_PLAN)
    try:
        for q, m in enumerate(models):
            r = configs.stream_res(cfg, cfg["queries"][q][1])
            G.gemel_register_model(ctx, m, _zero_params(m), q, r, r)
        seen = []

        def spy(c):
            seen.append([tuple(map(tuple, g["members"])) for g in c])
            return retrain(c)
        att, saved = G.gemel_incremental_merge(ctx, spy)
        assert [(a["group"], a["n_members"], a["ok"], a["bytes"]) for a in att] == \
            [(e["group"], len(e["members"]), e["ok"], e["bytes"]) for e in ref_log]
        assert saved == om.bytes_saved(models, ref_cfg) == G.gemel_stats(ctx)["bytes_saved"]
        # the library showed the oracle the same running configurations
        assert seen[-1][:-1] == [tuple(map(tuple, g["members"])) for g in ref_cfg][:len(seen[-1]) - 1]
    finally:
        G.gemel_destroy(ctx)


def test_library_errors():
    models = [zoo.build("tiny_a"), zoo.build("tiny_b")]
    ctx = G.gemel_create(flags=G.FLAG_DRY_PLAN)
    try:
        for q, m in enumerate(models):
            G.gemel_register_model(ctx, m, _zero_params(m), q, 32, 32)
        with pytest.raises(ZeroDivisionError):       # a failing callback aborts cleanly
            G.gemel_incremental_merge(ctx, lambda c: 1 / 0)
        G.gemel_apply_merge(ctx, [{"members": [(0, 0), (1, 0)], "source": 0}])
        with pytest.raises(G.GemelError) as e:      # needs an unmerged workload
            G.gemel_incremental_merge(ctx, lambda c: True)
        assert e.value.code == G.E_STATE
    finally:
        G.gemel_destroy(ctx)
