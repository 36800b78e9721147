"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Gate 1 (every config, including the exact bench configurations): per stored
value, teacher-forced -- the oracle layer applied to the device's own bf16
inputs, elementwise; an element above the relative gate is admitted only inside
the sqrt(K) fp32-accumulation bound of its GEMM, and at most a 1e-6 fraction of
the compared elements may be admitted (tests/gpu_util.py, reading R8).
Gate 2: end to end against the oracle in bf16-storage emulation -- elementwise
for cfg1 (4 param layers); for the deep free-running chains rare fp32-vs-fp64
rounding flips of stored bf16 values compound, so that gate is normwise
(max error <= 2e-2 x max |logit|, R8).  Merge configurations come from the
oracle (oracle.merge), never from the library.  Merge invariant: merged ==
unmerged-with-copied-weights, bitwise on the GPU.
Tolerance (north_star): max |gpu - oracle| / (|oracle| + 1e-3) <= 2e-2.
"""
import numpy as np
import pytest
import torch

from oracle import merge as om
from tests.gpu_util import TOL, make_queries, normwise_err, oracle_outputs, rel_err, teacher_forced
from workloads import configs, synth

pytestmark = pytest.mark.gpu


def _merge_cfg(models, merge):
    """The oracle's merge configuration: none / full (every signature class) / cross."""
    if merge == "none":
        return []
    groups = om.find_shareable(models)
    return om.full_merge(groups) if merge == "full" else om.cross_model_groups(groups)


def _run(models, params, names_streams, res, batch, merge, cfg_seed, engine_kw=None):
    from paper_2201_07705_b200.engine import MergedWorkload
    queries = [(m, p, s) for m, p, s in zip(models, params, names_streams)]
    wl = MergedWorkload(queries, res, batch, merge=_merge_cfg(models, merge), **(engine_kw or {}))
    frames_np = {s: synth.frames(cfg_seed, s, batch, res[0], res[1]) for s in sorted(set(names_streams))}
    frames = {s: torch.from_numpy(f).cuda() for s, f in frames_np.items()}
    outs = wl.alloc_outputs()
    wl.infer(frames, outs)
    torch.cuda.synchronize()
    return wl, frames_np, {m: o.cpu().numpy().astype(np.float64) for m, o in outs.items()}


@pytest.mark.parametrize("merge", ["full", "none"])
def test_cfg1_end_to_end(merge):
    """Free-running end to end.  Elementwise gate against the oracle in
    bf16-storage emulation (the device stores bf16 activations by design,
    DESIGN.md reading R7); against pure fp64 the storage rounding alone exceeds
    the 1e-3 floor on near-zero logits, so that comparison is normwise."""
    models, params = make_queries(1, ["tiny_a", "tiny_b"])
    wl, fr, outs = _run(models, params, [0, 1], (32, 32), 2, merge, 1)
    ref = oracle_outputs(models, params, wl.merge_config, [fr[0], fr[1]], emulate_bf16=True)
    ref64 = oracle_outputs(models, params, wl.merge_config, [fr[0], fr[1]])
    for mid in range(2):
        assert rel_err(outs[mid], ref[mid]) <= TOL
        assert np.abs(outs[mid] - ref64[mid]).max() <= TOL * np.abs(ref64[mid]).max()
    if merge == "full":
        assert wl.bytes_saved == 10176
        assert wl.plan["n_union_problems"] == 2       # conv0 and conv1 run once over both streams


def test_cfg1_teacher_forced():
    models, params = make_queries(1, ["tiny_a", "tiny_b"])
    wl, fr, _ = _run(models, params, [0, 1], (32, 32), 2, "full", 1)
    mp = om.merged_params(models, params, wl.merge_config)
    for mid in range(2):
        teacher_forced(wl.read_value, mid, models[mid], mp[mid], fr[mid]).check(mid)


def test_merged_equals_unmerged_with_copied_weights_bitwise():
    models, params = make_queries(1, ["tiny_a", "tiny_b"])
    wl_m, _, out_m = _run(models, params, [0, 1], (32, 32), 2, "full", 1)
    copied = om.merged_params(models, params, wl_m.merge_config)
    wl_u, _, out_u = _run(models, copied, [0, 1], (32, 32), 2, "none", 1)
    assert wl_u.plan["n_union_problems"] == 0
    for mid in range(2):
        np.testing.assert_array_equal(out_m[mid], out_u[mid])


def test_cfg2_small_teacher_forced():
    """ResNet-18/34/50 (cfg2 architectures) at 64x64, B=2: every stored value."""
    names = ["resnet18", "resnet34", "resnet50"]
    models, params = make_queries(2, names)
    wl, fr, outs = _run(models, params, [0, 1, 2], (64, 64), 2, "full", 2)
    assert wl.plan["n_union_problems"] > 0
    mp = om.merged_params(models, params, wl.merge_config)
    for mid in range(3):
        teacher_forced(wl.read_value, mid, models[mid], mp[mid], fr[mid]).check(names[mid])
    ref = oracle_outputs(models, params, wl.merge_config, [fr[0], fr[1], fr[2]], emulate_bf16=True)
    for mid in range(3):
        assert normwise_err(outs[mid], ref[mid]) <= TOL, names[mid]


def test_cfg2_full_size_sampled():
    """cfg2 in bench.py's launch configuration (224x224, B=8 per stream, cross merge):
    logits of sampled frames end to end against the oracle in bf16-storage emulation,
    frame by frame (Gate 2, normwise)."""
    names = ["resnet18", "resnet34", "resnet50"]
    models, params = make_queries(2, names)
    wl, fr, outs = _run(models, params, [0, 1, 2], (224, 224), 8, "cross", 2)
    mp = om.merged_params(models, params, wl.merge_config)
    from oracle import model as omodel
    for mid in range(3):
        for f in (0, 7):
            ref = omodel.run(models[mid], mp[mid], fr[mid][f:f + 1], emulate_bf16=True)[-1]
            assert normwise_err(outs[mid][f:f + 1], ref) <= TOL, (names[mid], f)


def test_cfg3_vgg_small_teacher_forced():
    """VGG-16/19 pair (cfg3 architectures) at 32x32: exercises 2x2 pools, the
    identity-replicating adaptive pool and the 25088-wide fc6 GEMM."""
    names = ["vgg16", "vgg19"]
    models, params = make_queries(3, names)
    wl, fr, outs = _run(models, params, [0, 1], (32, 32), 2, "full", 3)
    mp = om.merged_params(models, params, wl.merge_config)
    for mid in range(2):
        teacher_forced(wl.read_value, mid, models[mid], mp[mid], fr[mid]).check(names[mid])


def test_split_k_path_teacher_forced(monkeypatch):
    """Deterministic split-K (off by default) on the ResNets at 64x64: every
    stored value teacher-forced, and bitwise equal logits across two runs."""
    monkeypatch.setenv("GEMEL_MAX_SPLIT", "8")
    names = ["resnet18", "resnet50"]
    models, params = make_queries(2, names)
    wl, fr, outs = _run(models, params, [0, 1], (64, 64), 2, "full", 2)
    mp = om.merged_params(models, params, wl.merge_config)
    for mid in range(2):
        teacher_forced(wl.read_value, mid, models[mid], mp[mid], fr[mid]).check(names[mid])
    _, _, outs2 = _run(models, params, [0, 1], (64, 64), 2, "full", 2)
    for mid in range(2):
        np.testing.assert_array_equal(outs[mid], outs2[mid])


@pytest.mark.parametrize("names,res", [(("tiny_yolov3", "tiny_yolov3"), 416), (("yolov3", "yolov3"), 256),
                                       (("ssd300", "ssd300"), 300)])
def test_detector_teacher_forced_and_end_to_end(names, res):
    """YOLOv3 / Tiny-YOLOv3 pairs (cfg4/cfg5 detector family), cross-model merge
    (every layer of one model shares the other's weights; merging all 8 residual
    blocks of a stage into one weight would explode random-init activations): every
    stored value teacher-forced (darknet shortcut, route concat + fused nearest
    upsample, the 2x2 stride-1 darknet pool, the decode itself -- the decoded
    boxes against the oracle decode of the device's own head outputs -- and the
    top-100 selection, bit-exact on the device's own detection row), then end
    to end against the oracle in bf16-storage emulation on each head's raw output
    t (the detector's "logits").  Free-running bf16 chains drift chaotically
    (rounding flips spread layer by layer: tools/debug_yolo.py shows 0% -> 57% of
    elements differing by 1 ulp at ~0.5% normwise), and sigmoid/exp of the decode
    only re-scale that drift, so the end-to-end gate is normwise on t (R8)."""
    from oracle import model as omodel
    models, params = make_queries(4, list(names))
    wl, fr, outs = _run(models, params, [0, 1], (res, res), 2, "cross", 4)
    assert wl.plan["n_union_problems"] > 0
    assert all(len({m for m, _ in g["members"]}) == len(g["members"]) for g in wl.merge_config)
    mp = om.merged_params(models, params, wl.merge_config)
    for mid in range(2):
        errs = teacher_forced(wl.read_value, mid, models[mid], mp[mid], fr[mid]).check(names[mid])
        L = models[mid]
        assert len(L) - 4 in errs and L[len(L) - 4]["op"] == "concat"   # the decoded detection row was compared
        assert errs[len(L) - 2] == 0.0               # top candidates of the device's own rows: bit-exact
        assert errs[len(L) - 1] == 0.0               # final NMS detections: the oracle's decisions
    for mid in range(2):
        layers = models[mid]
        ref_all = omodel.run(layers, mp[mid], fr[mid], emulate_bf16=True)
        assert outs[mid].shape == ref_all[-1].shape
        for h in [j for l in layers if l["op"] in ("yolo", "ssd_decode") for j in l["in"]]:
            g = wl.read_value(mid, h).transpose(0, 3, 1, 2).astype(np.float64)
            assert normwise_err(g, ref_all[h]) <= TOL, (names[mid], h)


@pytest.mark.parametrize("names,res,frac,merge,source", [(("vgg16", "vgg19"), 32, 0.8, "none", "host"),
                                                         (("resnet18", "resnet34", "resnet50"), 64, 0.4, "none", "host"),
                                                         (("vgg16", "vgg19", "vgg16"), 32, 0.32, "cross", "host"),
                                                         (("vgg16", "vgg19"), 32, 0.8, "none", "peer")])
def test_weight_swap_matches_oracle_and_resident(names, res, frac, merge, source):
    """Budget mode: weights above the HBM budget stream every
    step from pinned host memory (or a peer GPU's HBM, N4) through the ring (copy stream, one launch ahead,
    inside the captured graph).  Every stored value of the swapped run is checked
    teacher-forced against the ORACLE, then against the all-resident run bitwise over
    several steps (ring slots are refilled every step)."""
    from oracle import plan as oplan
    from paper_2201_07705_b200 import gemel as G
    models, params = make_queries(3, list(names))
    budget = int(sum(om.param_bytes(l) for m in models for l in m) * frac)
    sids = list(range(len(names)))
    # "peer": weights above the budget paged from GPU memory (N4; the next GPU when there is
    # one, else this GPU's own HBM) instead of pinned host memory
    kw = {"weight_budget": budget}
    if source == "peer":
        kw.update(weight_source="peer", source_device=(torch.cuda.current_device() + 1) % torch.cuda.device_count())
    wl_s, fr, out_s = _run(models, params, sids, (res, res), 2, merge, 3, kw)
    assert wl_s.plan["n_swapped"] > 0 and wl_s.plan["weight_arena_bytes"] <= budget
    assert oplan.validate_swap(G.gemel_plan_dump(wl_s.ctx), budget)
    mp = om.merged_params(models, params, wl_s.merge_config)
    for mid in range(len(names)):
        teacher_forced(wl_s.read_value, mid, models[mid], mp[mid], fr[mid]).check((names[mid], "swapped"))
    wl_r, _, out_r = _run(models, params, sids, (res, res), 2, merge, 3)
    for mid in range(len(names)):
        np.testing.assert_array_equal(out_s[mid], out_r[mid])
    frames = {s: torch.from_numpy(f).cuda() for s, f in fr.items()}
    outs = wl_s.alloc_outputs()
    for _ in range(3):
        wl_s.infer(frames, outs)
    torch.cuda.synchronize()
    for mid in range(len(names)):
        np.testing.assert_array_equal(outs[mid].cpu().numpy().astype(np.float64), out_r[mid])


def test_mixed_resolution_streams_union_stems():
    """Streams at different resolutions (cfg5 mixes 224/300/416): a first conv over the
    ingest-written im2col rows unions across resolutions (rows are independent), the
    rest share weights only.  Every stored value teacher-forced."""
    from paper_2201_07705_b200.engine import MergedWorkload
    names = ["resnet18", "resnet18"]
    models, params = make_queries(2, names)
    res = {0: (64, 64), 1: (96, 96)}
    wl = MergedWorkload([(m, p, s) for s, (m, p) in enumerate(zip(models, params))], res, 2,
                        merge=_merge_cfg(models, "cross"))
    assert wl.plan["n_union_problems"] >= 1
    fr = {s: synth.frames(2, s, 2, *res[s]) for s in res}
    outs = wl.alloc_outputs()
    wl.infer({s: torch.from_numpy(f).cuda() for s, f in fr.items()}, outs)
    torch.cuda.synchronize()
    mp = om.merged_params(models, params, wl.merge_config)
    for mid in range(2):
        teacher_forced(wl.read_value, mid, models[mid], mp[mid], fr[mid]).check(mid)


@pytest.mark.parametrize("res", [64, 128])
def test_frcnn_teacher_forced_and_trunk_end_to_end(res):
    """Faster R-CNN R50-FPN pair (cfg4's second family), cross-model merge: every stored
    value teacher-forced -- FPN (lateral 1x1 + materialised nearest x2 top-down as the
    GEMM residual), the tied RPN head (one weight, 5 levels, each level a union over
    both models), the per-level RPN stage (top-1000 selection bit-exact on the device's
    own logits, boxes, NMS keep flags), the cross-level proposal merge, MultiScaleRoIAlign
    on the device's proposals and bf16 maps, the box head on M = frames x 1000 rows, the
    box decode + softmax and the top-100 selection (bit-exact).  At 64x64 fewer than
    1000 proposals survive (padded rows).  End to end (bf16-storage emulation): the
    FPN maps and RPN heads normwise (R8; the discrete stages are judged teacher-forced)."""
    from oracle import model as omodel
    models, params = make_queries(4, ["frcnn_r50_fpn", "frcnn_r50_fpn"])
    wl, fr, outs = _run(models, params, [0, 1], (res, res), 2, "cross", 4)
    assert wl.plan["n_union_problems"] > 0
    mp = om.merged_params(models, params, wl.merge_config)
    layers = models[0]
    last = len(layers) - 1
    for mid in range(2):
        errs = teacher_forced(wl.read_value, mid, models[mid], mp[mid], fr[mid]).check(mid)
        assert errs[last] == 0.0
        for op in ("rpn_level", "rpn_merge", "roi_align", "box_post"):
            assert any(layers[i]["op"] == op for i in errs), op
        props = wl.read_value(mid, next(i for i, l in enumerate(layers) if l["op"] == "rpn_merge")).reshape(2, -1, 5)
        if res == 64:
            assert props[:, :, 4].sum(axis=1).min() < 1000
    for mid in range(2):
        ref_all = omodel.run(layers, mp[mid], fr[mid], emulate_bf16=True)
        heads = [j for l in layers if l["op"] == "rpn_level" for j in l["in"]]
        maps = [layers[layers[layers[h]["in"][0]]["in"][0]]["in"][0] for h in heads[::2]]
        for h in heads + maps:
            g = wl.read_value(mid, h).transpose(0, 3, 1, 2).astype(np.float64)
            assert normwise_err(g, ref_all[h]) <= TOL, (mid, h, layers[h]["op"])


def test_cfg4_full_size_detector_stages_sampled():
    """cfg4 in the launch configuration bench.py times (4x YOLOv3 + 4x Faster R-CNN at
    608x608, B=4, cross merge): for one Faster R-CNN query, every detector stage against
    the oracle applied to the device's own inputs -- each RPN level (top-1000 of up to
    69 312 anchors bit-exact, boxes, NMS keep flags), the proposal merge (exact),
    MultiScaleRoIAlign on 64 sampled proposals per frame, the box decode + softmax (all
    rows) and the top-100 (exact); plus one YOLO query's detection row and top-100.
    (The trunks are covered end to end at 64-416 px; an fp64 trunk at 608 is ~140
    GFLOP per frame.)"""
    from oracle import ops
    cfg = configs.CONFIGS[4]
    names = [n for n, _ in cfg["queries"]]
    models, params = make_queries(4, names)
    sids = [s for _, s in cfg["queries"]]
    wl, fr, outs = _run(models, params, sids, (608, 608), 4, "cross", 4)
    mid = names.index("frcnn_r50_fpn")
    L = models[mid]

    def nchw(m, i):
        return wl.read_value(m, i).transpose(0, 3, 1, 2).astype(np.float64)

    def flat(m, i, n):
        v = wl.read_value(m, i)
        return v.reshape(v.shape[0], -1)[:, :n].astype(np.float64)

    lv = [i for i, l in enumerate(L) if l["op"] == "rpn_level"]
    rows = []
    for i in lv:
        l = L[i]
        A = len(l["ratios"])
        ref = ops.rpn_level(nchw(mid, l["in"][0])[:, :A], nchw(mid, l["in"][1])[:, :4 * A], l["size"], l["ratios"],
                            l["pre_n"], l["nms"], l["min_size"], (608, 608))
        got = flat(mid, i, ref.shape[1])
        r6, g6 = ref.reshape(4, -1, 6), got.reshape(4, -1, 6)
        np.testing.assert_array_equal(g6[..., 4], r6[..., 4])             # selection and order: exact
        # fp32 decode of pixel coordinates (<= 608, pre-clip widths up to ~3e4): a few fp32 ulps
        assert np.abs(g6[..., :4] - r6[..., :4]).max() <= 1e-3
        assert (g6[..., 5] != r6[..., 5]).sum() <= 2, i                   # NMS decisions (fp32 vs fp64 IoU ties)
        rows.append(got)
    m = next(i for i, l in enumerate(L) if l["op"] == "rpn_merge")
    props = flat(mid, m, 5000)
    np.testing.assert_array_equal(props, ops.rpn_merge(rows, 1000))
    r = next(i for i, l in enumerate(L) if l["op"] == "roi_align")
    maps = [nchw(mid, j) for j in L[r]["in"][1:]]
    g = wl.read_value(mid, r).astype(np.float64)                          # [4 * 1000, 7, 7, 256]
    rng = np.random.default_rng(0)
    for f in range(4):
        pick = np.sort(rng.choice(1000, 64, replace=False))
        sub = props[f].reshape(1000, 5)[pick].reshape(1, -1)
        refr = ops.multiscale_roi_align([mm[f:f + 1] for mm in maps], sub, 7, 2, (224, 4), (608, 608))
        assert rel_err(g[f * 1000 + pick].transpose(0, 3, 1, 2), refr) <= TOL, f
    b = next(i for i, l in enumerate(L) if l["op"] == "box_post")
    refb = ops.box_post(flat(mid, L[b]["in"][0], 91), flat(mid, L[b]["in"][1], 364), props, 91,
                        (10.0, 10.0, 5.0, 5.0), (608, 608))
    gotb = flat(mid, b, refb.shape[1])
    g6, r6 = gotb.reshape(4, -1, 6), refb.reshape(4, -1, 6)
    assert np.abs(g6[..., :4] - r6[..., :4]).max() <= 1e-3                # decoded boxes (pixels)
    assert rel_err(g6[..., 4], r6[..., 4]) <= 1e-4                         # softmax probabilities
    np.testing.assert_array_equal(g6[..., 5], r6[..., 5])                  # class labels
    _check_final_detections(wl, mid, L, outs[mid])
    ym = names.index("yolov3")
    Y = models[ym]
    det = len(Y) - 4
    sizes = []
    for h in Y[det]["in"]:
        y = Y[h]
        F = len(y["anchors"]) * (5 + y["classes"])
        sizes.append((h, ops.yolo_decode(nchw(ym, y["in"][0])[:, :F], y["anchors"], y["classes"], (608, 608))))
    n_row = sum(v.shape[1] for _, v in sizes)
    row = flat(ym, det, n_row)
    off = 0
    for h, refy in sizes:
        assert rel_err(row[:, off:off + refy.shape[1]], refy) <= TOL, h
        off += refy.shape[1]
    _check_final_detections(wl, ym, Y, outs[ym])


def _check_final_detections(wl, mid, L, out):
    """N2 tail on the device's own inputs: det_cand rows (decisions at the threshold),
    the top-k candidates (bit-exact) and the NMS detections (the oracle's decisions)
    equal the model output."""
    from oracle import ops
    from tests.gpu_util import det_stage_err
    n = len(L)
    assert [L[i]["op"] for i in range(n - 3, n)] == ["det_cand", "topk", "det_nms"]

    def flat(i):
        v = wl.read_value(mid, i)
        return v.reshape(v.shape[0], -1).astype(np.float64)
    row, cand, top, fin = flat(n - 4), flat(n - 3), flat(n - 2), flat(n - 1)
    lc, lt, ln = L[n - 3], L[n - 2], L[n - 1]
    ref_c = ops.det_candidates(row[:, :cand.shape[1] // 6 * lc["fields"]], lc["fmt"], lc["fields"],
                               lc["score_thresh"], lc["min_size"])
    assert det_stage_err("det_cand", cand, ref_c, lc) == 0.0
    np.testing.assert_array_equal(top, ops.topk_rows(cand, lt["k"], 6, 4))
    assert det_stage_err("det_nms", fin, ops.det_nms(top, ln["iou"], ln["max_det"]), dict(ln, _top=top)) == 0.0
    np.testing.assert_array_equal(np.asarray(out, np.float64).reshape(fin.shape), fin)
    assert (fin.reshape(fin.shape[0], -1, 6)[..., 4] >= 0).sum() > 0   # something was detected


@pytest.mark.parametrize("cfg_id,picks", [(3, [0, 1]), (5, [0, 5, 13, 14, 21, 26])])
def test_full_size_configs_sampled(cfg_id, picks):
    """cfg3 (6 VGGs, B=8) and cfg5 (the 32-stream mix, B=4) in the launch configuration
    bench.py times, cross merge: for sampled queries (cfg5: R18, R50, R152, VGG11,
    VGG19 and Tiny-YOLOv3's two heads) and frames 0 and B-1, the model outputs end to
    end against the oracle in bf16-storage emulation (normwise, reading R8)."""
    from oracle import model as omodel
    cfg = configs.CONFIGS[cfg_id]
    names = [n for n, _ in cfg["queries"]]
    sids = [s for _, s in cfg["queries"]]
    models, params = make_queries(cfg_id, names)
    from paper_2201_07705_b200.engine import MergedWorkload
    res = {s: (configs.stream_res(cfg, s),) * 2 for s in sids}
    wl = MergedWorkload([(m, p, s) for m, p, s in zip(models, params, sids)], res, cfg["batch"],
                        merge=_merge_cfg(models, "cross"))
    fr = {s: synth.frames(cfg_id, s, cfg["batch"], res[s][0], res[s][1]) for s in sids}
    outs = wl.alloc_outputs()
    wl.infer({s: torch.from_numpy(f).cuda() for s, f in fr.items()}, outs)
    torch.cuda.synchronize()
    mp = om.merged_params(models, params, wl.merge_config)
    B = cfg["batch"]
    for q in picks:
        layers = models[q]
        heads = [j for l in layers if l["op"] in ("yolo", "ssd_decode") for j in l["in"]]
        for f in (0, B - 1):
            vals = omodel.run(layers, mp[q], fr[sids[q]][f:f + 1], emulate_bf16=True)
            if heads:   # detector: its raw head outputs t (the decode is gated teacher-forced elsewhere)
                for h in heads:
                    g = wl.read_value(q, h)[f:f + 1].transpose(0, 3, 1, 2).astype(np.float64)
                    assert normwise_err(g[:, :vals[h].shape[1]], vals[h]) <= TOL, (names[q], h, f)
            else:
                got = outs[q][f:f + 1].cpu().numpy().astype(np.float64)
                assert normwise_err(got, vals[-1]) <= TOL, (names[q], f)
    wl.close()


@pytest.mark.parametrize("cfg_id", [2, 3, 4, 5])
def test_bench_config_teacher_forced_elementwise(cfg_id):
    """Gate 1 at the exact configurations bench.py times (configs.CONFIGS[cfg]: its
    models, streams, B and resolutions; cross merge from the oracle; bench.py's
    weight and frame seeds): for EVERY query, frames 0 and B-1, every value the
    device stores -- conv/linear chains, pools, concats, decodes, detector stages,
    top-100 -- against the oracle layer applied to the device's own inputs,
    elementwise (admissions capped and reported, tests/gpu_util.py)."""
    from paper_2201_07705_b200.engine import MergedWorkload
    from tests import gpu_util
    cfg = configs.CONFIGS[cfg_id]
    names = [n for n, _ in cfg["queries"]]
    sids = [s for _, s in cfg["queries"]]
    models, params = make_queries(cfg_id, names)
    merge = _merge_cfg(models, "cross")
    res = {s: (configs.stream_res(cfg, s),) * 2 for s in sids}
    B = cfg["batch"]
    wl = MergedWorkload([(m, p, s) for m, p, s in zip(models, params, sids)], res, B, merge=merge)
    fr = {s: synth.frames(cfg_id, s, B, res[s][0], res[s][1]) for s in sids}
    outs = wl.alloc_outputs()
    wl.infer({s: torch.from_numpy(f).cuda() for s, f in fr.items()}, outs)
    torch.cuda.synchronize()
    mp = om.merged_params(models, params, merge)
    admitted = total = 0
    for q in range(len(models)):
        rep = teacher_forced(wl.read_value, q, models[q], mp[q], fr[sids[q]], frames=(0, B - 1))
        rep.check((cfg["name"], q, names[q]))
        admitted += rep.admitted
        total += rep.total
    assert admitted <= 1e-5 * total, (admitted, total)   # aggregate over the config (measured <= 2.1e-6)
    wl.close()
