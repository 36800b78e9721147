"""Pins of the oracle's plan-side functions and the host
planner checked against them (dry plan, no GPU):

* oracle.plan.min_swap_bytes (exhaustive search) against closed forms; the
  library's resident-set selection against it on random <= 6-tensor instances;
* oracle.plan.validate_swap REJECTS each kind of broken residency plan;
* oracle.plan.lcs_length / scs_length against textbook values and brute force;
  the planner's GEMM problem count for two chains == the SCS length;
* oracle.merge.cross_model_groups against its closed form, and the library-side
  merge configuration (engine.cross_model_merge_config) equal to it.
"""
import copy
import itertools
import random
from collections import Counter

import pytest

from oracle import merge as om
from oracle import model as omodel
from oracle import plan as oplan
from workloads import configs, zoo

G = pytest.importorskip("paper_2201_07705_b200.gemel")
from tests.test_plan import _plan_budget, _zero_params  # noqa: E402

AL = 256


def _al(x):
    return (x + AL - 1) // AL * AL


# ---------------------------------------------------------------- minimal swap bytes
def test_min_swap_closed_forms():
    # everything fits: nothing streams
    assert oplan.min_swap_bytes([1000, 3000, 500], _al(1000) + _al(3000) + _al(500)) == 0
    # a single tensor either fits or cannot be double-buffered (its ring is 2x larger)
    assert oplan.min_swap_bytes([5000], _al(5000)) == 0
    assert oplan.min_swap_bytes([5000], _al(5000) - 1) is None
    # n equal tensors of aligned size s: k = A // s - 2 stay resident, n - k stream
    for n in range(1, 7):
        for A in range(2 * AL, (n + 3) * AL, AL // 2):
            got = oplan.min_swap_bytes([AL] * n, A)
            if n * AL <= A:
                assert got == 0
            else:
                k = A // AL - 2
                assert got == (n - max(k, 0)) * AL, (n, A, got)
    # one big + four small tensors, budget big + 3 small: streaming the big one needs a
    # 2 x big ring (> budget), so big stays resident with one small and three stream
    big, small = 10 * AL, AL
    assert oplan.min_swap_bytes([big, small, small, small, small], big + 3 * small) == 3 * small


def test_min_swap_bounds_random():
    rng = random.Random(7)
    for _ in range(200):
        sizes = [rng.randint(1, 20) * 100 for _ in range(rng.randint(1, 6))]
        A = rng.randint(0, sum(_al(s) for s in sizes) + 2 * AL)
        got = oplan.min_swap_bytes(sizes, A)
        tot = sum(_al(s) for s in sizes)
        if got is None:     # infeasible: not all resident, and not all streamed either
            assert tot > A and 2 * max(_al(s) for s in sizes) > A
            continue
        assert got >= max(0, sum(sizes) - A - 256 * len(sizes))   # lower bound: W - budget (modulo alignment)
        # monotone in the budget
        g2 = oplan.min_swap_bytes(sizes, A + AL)
        assert g2 is not None and g2 <= got


def _chain(channels):
    layers, prev = [], -1
    for i in range(len(channels) - 1):
        layers.append({"op": "conv", "in": [prev], "cin": channels[i], "cout": channels[i + 1], "k": (1, 1),
                       "s": (1, 1), "p": (0, 0), "d": (1, 1), "groups": 1, "bias": False})
        prev = len(layers) - 1
    return layers


def test_library_resident_set_is_minimal():
    """The planner's pinned set streams the fewest bytes: equal to the exhaustive
    optimum on random chains of 2-6 weights (each a 1x1 conv GEMM node whose fp32
    scale/shift epilogue vectors stay resident, reading R14), with a valid plan."""
    rng = random.Random(0)
    checked = 0
    for _ in range(40):
        ch = [3] + [8 * rng.randint(1, 40) for _ in range(rng.randint(2, 6))]
        m = _chain(ch)
        epi = sum(2 * _al(l["cout"] * 4) for l in m)
        ctx0 = G.gemel_create(flags=G.FLAG_DRY_PLAN)
        G.gemel_register_model(ctx0, m, _zero_params(m), 0, 8, 8)
        G.gemel_plan(ctx0, [1])
        sizes = [w["bytes"] for w in G.gemel_plan_dump(ctx0)["swap"]["weights"]]
        G.gemel_destroy(ctx0)
        budget = epi + rng.randint(0, sum(_al(s) for s in sizes))
        opt = oplan.min_swap_bytes(sizes, budget - epi)
        ctx = G.gemel_create(flags=G.FLAG_DRY_PLAN, weight_budget_bytes=budget)
        G.gemel_register_model(ctx, m, _zero_params(m), 0, 8, 8)
        try:
            info = G.gemel_plan(ctx, [1])
            lib = info["swap_bytes_per_step"]
            assert oplan.validate_swap(G.gemel_plan_dump(ctx), budget)
        except G.GemelError as e:
            assert e.code == G.E_NOMEM
            lib = None
        finally:
            G.gemel_destroy(ctx)
        assert lib == opt, (sizes, budget - epi, lib, opt)
        checked += lib is not None and lib > 0
    assert checked >= 5


# ---------------------------------------------------------------- validate_swap rejects
@pytest.fixture(scope="module")
def swap_dump():
    _, _, info, dump, budget = _plan_budget(("vgg16", "vgg19", "vgg16"), 224, 2, "none", 0.5)
    assert info["n_swapped"] >= 2
    assert oplan.validate_swap(dump, budget)
    return dump, budget


def _streamed(d):
    return [w for w in d["swap"]["weights"] if w["swapped"]]


def test_validate_swap_rejects_arena_over_budget(swap_dump):
    dump, budget = swap_dump
    with pytest.raises(AssertionError):
        oplan.validate_swap(dump, dump["swap"]["weight_arena_bytes"] - 1)


def test_validate_swap_rejects_copy_after_first_use(swap_dump):
    dump, budget = swap_dump
    bad = copy.deepcopy(dump)
    w = _streamed(bad)[0]
    w["wait_launch"] = w["first_launch"]
    with pytest.raises(AssertionError):
        oplan.validate_swap(bad, budget)


def test_validate_swap_rejects_overlapping_live_slots(swap_dump):
    """Two streamed tensors whose lifetimes overlap placed in the same slot."""
    dump, budget = swap_dump
    bad = copy.deepcopy(dump)
    s = sorted(_streamed(bad), key=lambda w: w["copy_order"])
    a, b = s[0], s[1]
    b["offset"] = a["offset"]                       # same slot ...
    b["wait_launch"] = min(a["last_launch"], b["first_launch"]) - 1   # ... refilled while a is still read
    with pytest.raises(AssertionError):
        oplan.validate_swap(bad, budget)


def test_validate_swap_rejects_slot_overwritten_while_read(swap_dump):
    dump, budget = swap_dump
    bad = copy.deepcopy(dump)
    s = sorted(_streamed(bad), key=lambda w: w["copy_order"])
    pair = next(((a, b) for i, a in enumerate(s) for b in s[i + 1:]
                 if a["offset"] < b["offset"] + b["bytes"] and b["offset"] < a["offset"] + a["bytes"]), None)
    if pair is None:   # no slot reuse in this plan: force one
        a, b = s[0], s[1]
        b["offset"] = a["offset"]
    else:
        a, b = pair
    b["wait_launch"] = a["last_launch"] - 1
    with pytest.raises(AssertionError):
        oplan.validate_swap(bad, budget)


def test_validate_swap_rejects_pinned_overlap_and_ring_escape(swap_dump):
    dump, budget = swap_dump
    pinned = [w for w in dump["swap"]["weights"] if not w["swapped"]]
    assert len(pinned) >= 2
    bad = copy.deepcopy(dump)
    p = [w for w in bad["swap"]["weights"] if not w["swapped"]]
    p[1]["offset"] = p[0]["offset"]                  # two resident weights on the same bytes
    with pytest.raises(AssertionError):
        oplan.validate_swap(bad, budget)
    bad = copy.deepcopy(dump)
    p = [w for w in bad["swap"]["weights"] if not w["swapped"]]
    p[0]["offset"] = bad["swap"]["ring_off"]         # a resident weight inside the ring
    with pytest.raises(AssertionError):
        oplan.validate_swap(bad, budget)
    bad = copy.deepcopy(dump)
    _streamed(bad)[0]["offset"] = bad["swap"]["ring_off"] + bad["swap"]["ring_bytes"]   # slot past the ring
    with pytest.raises(AssertionError):
        oplan.validate_swap(bad, budget)


def test_validate_swap_rejects_wrong_swap_bytes_and_lifetime(swap_dump):
    dump, budget = swap_dump
    bad = copy.deepcopy(dump)
    bad["swap"]["swap_bytes"] += 1
    with pytest.raises(AssertionError):
        oplan.validate_swap(bad, budget)
    bad = copy.deepcopy(dump)
    _streamed(bad)[0]["first_launch"] += 1
    with pytest.raises(AssertionError):
        oplan.validate_swap(bad, budget)


# ---------------------------------------------------------------- LCS / SCS
def test_lcs_scs_textbook():
    eq = lambda x, y: x == y  # noqa: E731
    assert oplan.lcs_length("ABCBDAB", "BDCABA", eq) == 4     # CLRS 15.4
    assert oplan.scs_length("ABCBDAB", "BDCABA", eq) == 9
    assert oplan.lcs_length("", "ABC", eq) == 0 and oplan.scs_length("", "ABC", eq) == 3
    assert oplan.scs_length("AGGTAB", "GXTXAYB", eq) == 9


def _is_subseq(s, t):
    it = iter(t)
    return all(c in it for c in s)


def test_lcs_scs_brute_force():
    rng = random.Random(3)
    eq = lambda x, y: x == y  # noqa: E731
    for _ in range(60):
        a = "".join(rng.choice("xy") for _ in range(rng.randint(0, 5)))
        b = "".join(rng.choice("xy") for _ in range(rng.randint(0, 5)))
        lcs = max(len(s) for r in range(len(a) + 1) for s in ("".join(c) for c in itertools.combinations(a, r))
                  if _is_subseq(s, b))
        assert oplan.lcs_length(a, b, eq) == lcs
        L = max(len(a), len(b))
        while not any(_is_subseq(a, "".join(t)) and _is_subseq(b, "".join(t))
                      for t in itertools.product("xy", repeat=L)):
            L += 1
        assert oplan.scs_length(a, b, eq) == L, (a, b)


@pytest.mark.parametrize("names", [("vgg16", "vgg19"), ("vgg11", "vgg13"), ("vgg16", "vgg16"), ("vgg11", "vgg19"),
                                   ("alexnet", "vgg16")])
def test_two_chain_union_is_scs(names):
    """Two chain models (VGG/AlexNet) under the cross-model merge: the planner's GEMM
    problems are the shortest common supersequence of the two GEMM-layer sequences,
    where two layers union iff they are bound to one weight AND see the same input
    shape (one TMA map over their concatenated batch) -- exact DP (§8(c)(iii))."""
    models = [zoo.build(n) for n in names]
    cfg = om.cross_model_groups(om.find_shareable(models))
    ctx = G.gemel_create(flags=G.FLAG_DRY_PLAN)
    for i, m in enumerate(models):
        G.gemel_register_model(ctx, m, _zero_params(m), i, 224, 224)
    if cfg:
        G.gemel_apply_merge(ctx, cfg)
    info = G.gemel_plan(ctx, [2, 2])
    G.gemel_destroy(ctx)
    grp = {tuple(mm): gi for gi, g in enumerate(cfg) for mm in g["members"]}
    seqs = []
    for mi, m in enumerate(models):
        shp = omodel.shapes(m, (224, 224))
        seqs.append([((mi, p), (3, 224, 224) if l["in"][0] < 0 else shp[l["in"][0]])
                     for p, l in enumerate(m) if l["op"] in ("conv", "linear")])

    def match(a, b):
        return a[0] in grp and grp[a[0]] == grp.get(b[0]) and a[1] == b[1]
    assert info["n_gemm_problems"] == oplan.scs_length(seqs[0], seqs[1], match)


# ---------------------------------------------------------------- cross-model groups
@pytest.mark.parametrize("cfg_id", [1, 2, 3, 4, 5])
def test_cross_model_groups_closed_form(cfg_id):
    """Each group holds <= 1 appearance per model and one signature; bytes saved
    = sum over signature classes of bytes * (sum_i c_i - max_i c_i), c_i = the class's
    appearances in model i (SURVEY.md §8(c)(iii) independent recomputation)."""
    cfg = configs.CONFIGS[cfg_id]
    models = [zoo.build(n) for n, _ in cfg["queries"]]
    groups = om.find_shareable(models)
    cross = om.cross_model_groups(groups)
    om.validate_merge(models, cross)
    for g in cross:
        assert len({m for m, _ in g["members"]}) == len(g["members"]) >= 2
    closed = 0
    for g in groups:
        c = Counter(m for m, _ in g["apps"])
        closed += g["per_bytes"] * (sum(c.values()) - max(c.values()))
    assert om.bytes_saved(models, cross) == closed
    if cfg_id == 1:
        assert closed == 10176        # SURVEY.md §8(c)(iii) cfg1 worked example


@pytest.mark.parametrize("cfg_id", [2, 3, 4, 5])
def test_engine_cross_config_equals_oracle(cfg_id):
    """The library side's merge configuration (from the library's find_shareable) is
    the oracle's, member for member (integer work: bit-exact)."""
    from paper_2201_07705_b200.engine import cross_model_merge_config
    cfg = configs.CONFIGS[cfg_id]
    models = [zoo.build(n) for n, _ in cfg["queries"]]
    ctx = G.gemel_create(flags=G.FLAG_DRY_PLAN)
    for q, m in enumerate(models):
        r = configs.stream_res(cfg, cfg["queries"][q][1])
        G.gemel_register_model(ctx, m, _zero_params(m), q, r, r)
    lib = cross_model_merge_config(G.gemel_find_shareable(ctx))
    G.gemel_destroy(ctx)
    ref = om.cross_model_groups(om.find_shareable(models))

    def norm(c):
        return sorted((tuple(tuple(x) for x in g["members"]), g["source"]) for g in c)
    assert norm(lib) == norm(ref)
