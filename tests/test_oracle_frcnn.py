"""Pins for the oracle's Faster R-CNN R50-FPN stages (oracle/ops.py: rpn_anchors,
box_decode, nms, rpn_level, rpn_merge, roi_align, multiscale_roi_align, box_post)
and the zoo model: torchvision (an independent implementation, fp64 on CPU)
stage by stage, closed forms and brute force."""
import math

import numpy as np
import pytest
import torch
import torchvision
from torchvision.models.detection import fasterrcnn_resnet50_fpn
from torchvision.models.detection.image_list import ImageList

from oracle import merge, model, ops
from workloads import synth, zoo


def _tv_frcnn(layers, params):
    net = fasterrcnn_resnet50_fpn(weights=None, weights_backbone=None, num_classes=91).double().eval()
    mods = [m for m in net.modules() if isinstance(m, (torch.nn.Conv2d, torch.nn.BatchNorm2d, torch.nn.Linear))]
    ours = [(l, p) for l, p in zip(layers, params) if merge.signature(l) is not None]
    assert len(mods) == len(ours) == 121
    with torch.no_grad():
        for m, (l, p) in zip(mods, ours):
            if l["op"] == "bn":
                assert isinstance(m, torch.nn.BatchNorm2d) and m.num_features == l["c"]
                for a, k in (("weight", "gamma"), ("bias", "beta"), ("running_mean", "mean"), ("running_var", "var")):
                    getattr(m, a).copy_(torch.from_numpy(p[k].astype(np.float64)))
            else:
                assert tuple(m.weight.shape) == p["w"].shape, (m, p["w"].shape)
                m.weight.copy_(torch.from_numpy(p["w"].astype(np.float64)))
                assert ("b" in p) == (m.bias is not None)
                if "b" in p:
                    m.bias.copy_(torch.from_numpy(p["b"].astype(np.float64)))
    return net


def test_frcnn_param_count_vs_torchvision():
    """121 param layers, torchvision's 41,808,406 parameters plus the
    53,120 BN running statistics; the RPN head is counted once (tied over 5 levels)."""
    layers = zoo.build("frcnn_r50_fpn")
    net = fasterrcnn_resnet50_fpn(weights=None, weights_backbone=None, num_classes=91)
    n_tv = sum(p.numel() for p in net.parameters())
    stats = sum(b.numel() for n, b in net.named_buffers() if "running" in n)
    assert n_tv == 41_808_406 and stats == 53_120
    assert sum(merge.param_count(l) for l in layers) == n_tv + stats
    assert sum(merge.signature(l) is not None for l in layers) == 121
    assert sum("tie" in l for l in layers) == 12              # 3 head convs x 4 more levels


@pytest.mark.parametrize("res", [64, 128])
def test_frcnn_stages_match_torchvision(res):
    """Whole model at res x res (N = 2): FPN maps, RPN proposals (count, order,
    values), MultiScaleRoIAlign features, box-head logits / deltas and the decoded
    (box, probability) rows, against torchvision's modules on the same weights.
    At 64x64 fewer than 1000 proposals survive NMS: the padded rows are checked."""
    layers = zoo.build("frcnn_r50_fpn")
    params = synth.params(layers, 41, 0)
    fr = synth.frames(41, 0, 2, res, res)
    vals = model.run(layers, params, fr)
    net = _tv_frcnn(layers, params)
    x = torch.from_numpy(ops.preprocess(fr))
    sizes = [(res, res)] * 2
    with torch.no_grad():
        feats = net.backbone(x)
        props, _ = net.rpn(ImageList(x, sizes), feats)
        bf = net.roi_heads.box_roi_pool(feats, props, sizes)
        h = net.roi_heads.box_head(bf)
        cl, br = net.roi_heads.box_predictor(h)
        boxes = net.roi_heads.box_coder.decode(br, props)
        scores = torch.softmax(cl, -1)
    pos = {op: [i for i, l in enumerate(layers) if l["op"] == op] for op in ("rpn_level", "rpn_merge", "roi_align",
                                                                               "box_post", "linear")}
    fpn_maps = [layers[p]["in"][0] for p in pos["rpn_level"]]   # P2..P6 via the RPN head inputs
    fpn_maps = [layers[layers[layers[m]["in"][0]]["in"][0]]["in"][0] for m in fpn_maps]
    for k, key in enumerate(["0", "1", "2", "3", "pool"]):
        ref = feats[key].numpy()
        np.testing.assert_allclose(vals[fpn_maps[k]], ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())
    pr = vals[pos["rpn_merge"][0]].reshape(2, -1, 5)
    counts = []
    for i in range(2):
        n = int(pr[i, :, 4].sum())
        counts.append(n)
        assert n == len(props[i])
        np.testing.assert_allclose(pr[i, :n, :4], props[i].numpy(), rtol=1e-9, atol=1e-9 * res)
        assert np.all(pr[i, n:] == 0)
    if res == 64:
        assert min(counts) < 1000                       # the padded-row case is exercised
    R = pr.shape[1]
    ra = vals[pos["roi_align"][0]].reshape(2, R, -1)
    rb = bf.numpy().reshape(sum(counts), -1)
    np.testing.assert_allclose(np.concatenate([ra[i, :counts[i]] for i in range(2)]), rb, rtol=1e-9,
                               atol=1e-9 * np.abs(rb).max())
    lg = vals[pos["linear"][2]].reshape(2, R, -1)
    np.testing.assert_allclose(np.concatenate([lg[i, :counts[i]] for i in range(2)]), cl.numpy(), rtol=1e-9,
                               atol=1e-9 * np.abs(cl.numpy()).max())
    det = vals[pos["box_post"][0]].reshape(2, R, 90, 6)
    off = 0
    for i in range(2):
        n = counts[i]
        b = torchvision.ops.clip_boxes_to_image(boxes[off:off + n], sizes[i]).numpy()
        np.testing.assert_allclose(det[i, :n, :, :4], b[:, 1:], rtol=1e-9, atol=1e-9 * res)
        np.testing.assert_allclose(det[i, :n, :, 4], scores[off:off + n, 1:].numpy(), rtol=1e-9, atol=1e-15)
        assert np.all(det[i, n:, :, 4] == -1.0)
        assert np.all(det[i, :, :, 5] == np.arange(1, 91))
        off += n
    top = vals[-2].reshape(2, 1024, 7)
    for i in range(2):   # the 1024 best (proposal, class) candidates (score > 0.011, sides >= 1e-2)
        r = det[i].reshape(-1, 6)
        ok = (r[:, 4] > 0.011) & (r[:, 2] - r[:, 0] >= 1e-2) & (r[:, 3] - r[:, 1] >= 1e-2)
        s = np.sort(r[ok, 4])[::-1][:1024]
        assert np.allclose(s, top[i, :len(s), 5]) and np.all(top[i, len(s):, 5] == -1.0 * (top[i, len(s):, 0] >= 0))


def test_anchors_vs_torchvision_anchor_generator():
    from torchvision.models.detection.anchor_utils import AnchorGenerator
    gen = AnchorGenerator(((32,), (64,), (128,), (256,), (512,)), ((0.5, 1.0, 2.0),) * 5)
    img = torch.zeros(1, 3, 96, 160, dtype=torch.float64)
    fm = [torch.zeros(1, 4, 96 // s, 160 // s, dtype=torch.float64) for s in (4, 8, 16, 32)]
    fm.append(torch.zeros(1, 4, 2, 3, dtype=torch.float64))       # P6-like: stride 96//2, 160//3
    ref = gen(ImageList(img, [(96, 160)]), fm)[0].numpy()
    ours = np.concatenate([ops.rpn_anchors(32 << k, (0.5, 1.0, 2.0), f.shape[2:], (96, 160)) for k, f in enumerate(fm)])
    np.testing.assert_array_equal(ours, ref)


def test_anchor_closed_form():
    """ratio 1: the square of side `size` centred on the stride grid point."""
    a = ops.rpn_anchors(64, (1.0,), (2, 3), (32, 48))
    assert a.shape == (6, 4)
    np.testing.assert_array_equal(a[4], [16 - 32, 16 - 32, 16 + 32, 16 + 32])    # y = 1, x = 1, stride 16


def test_box_decode_vs_torchvision_and_identity():
    from torchvision.models.detection._utils import BoxCoder
    g = np.random.default_rng(0)
    anc = np.cumsum(g.uniform(1, 50, (200, 4)), axis=1)
    d = g.normal(0, 2, (200, 4))
    for w in ((1.0, 1.0, 1.0, 1.0), (10.0, 10.0, 5.0, 5.0)):
        ref = BoxCoder(w).decode_single(torch.from_numpy(d), torch.from_numpy(anc)).numpy()
        np.testing.assert_allclose(ops.box_decode(d, anc, w), ref, rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(ops.box_decode(np.zeros((200, 4)), anc, (1, 1, 1, 1)), anc, rtol=1e-12)
    big = ops.box_decode(np.array([[0, 0, 100.0, 0]]), np.array([[0, 0, 10.0, 10.0]]), (1, 1, 1, 1))
    assert math.isclose(big[0, 2] - big[0, 0], 10 * 1000 / 16, rel_tol=1e-12)   # dw clamped at log(1000/16)


def test_nms_vs_torchvision_and_brute_force():
    g = np.random.default_rng(1)
    for trial in range(20):
        n = int(g.integers(1, 300))
        xy = g.uniform(0, 100, (n, 2))
        wh = g.uniform(0, 40, (n, 2)) * (g.uniform(size=(n, 1)) > 0.05)   # some zero-area boxes
        b = np.concatenate([xy, xy + wh], axis=1)
        s = np.round(g.uniform(0, 1, n), 2 if trial % 2 else 12)          # ties on odd trials
        thr = float(g.choice([0.3, 0.5, 0.7]))
        ours = ops.nms(b, s, thr)
        if trial % 2 == 0:
            assert ours == torchvision.ops.nms(torch.from_numpy(b), torch.from_numpy(s), thr).tolist()
        # brute force of the definition: a box is kept iff no kept box earlier in the
        # (score desc, index asc) order overlaps it with IoU > thr
        order = sorted(range(n), key=lambda i: (-s[i], i))
        kept = []
        for i in order:
            ok = True
            for j in kept:
                iw = max(0.0, min(b[i, 2], b[j, 2]) - max(b[i, 0], b[j, 0]))
                ih = max(0.0, min(b[i, 3], b[j, 3]) - max(b[i, 1], b[j, 1]))
                inter = iw * ih
                den = (b[i, 2] - b[i, 0]) * (b[i, 3] - b[i, 1]) + (b[j, 2] - b[j, 0]) * (b[j, 3] - b[j, 1]) - inter
                if den > 0 and inter / den > thr:
                    ok = False
                    break
            if ok:
                kept.append(i)
        assert ours == kept


def test_nms_special_cases():
    b = np.array([[0, 0, 10, 10]] * 3 + [[20, 20, 30, 30]], float)
    assert ops.nms(b, np.array([0.5, 0.9, 0.9, 0.1]), 0.7) == [1, 3]      # duplicates: first of the tie kept
    assert ops.nms(b[[0, 3]], np.array([0.2, 0.3]), 0.0) == [1, 0]           # disjoint: IoU 0 never > 0


@pytest.mark.parametrize("aligned_case", range(3))
def test_roi_align_vs_torchvision(aligned_case):
    g = np.random.default_rng(2 + aligned_case)
    C, H, W = 5, 13, 17
    f = g.normal(size=(C, H, W))
    scale = [0.25, 0.5, 1.0][aligned_case]
    xy = g.uniform(-20, 80, (60, 2))
    wh = g.uniform(0, 40, (60, 2))
    rois = np.concatenate([xy, xy + wh], axis=1)
    rois[:3] = [[0, 0, 0, 0], [1, 1, 1.5, 1.5], [-30, -30, -10, -10]]        # empty, sub-bin, outside
    ref = torchvision.ops.roi_align(torch.from_numpy(f)[None], [torch.from_numpy(rois)], 7, scale, 2,
                                    aligned=False).numpy()
    np.testing.assert_allclose(ops.roi_align(f, rois, 7, scale, 2), ref, rtol=1e-12, atol=1e-12)


def test_roi_align_closed_forms():
    """constant map -> constant (rois inside); ramp f = x -> mean sample x (bilinear
    is exact on linear functions)."""
    C, H, W = 2, 20, 20
    f = np.full((C, H, W), 3.25)
    np.testing.assert_allclose(ops.roi_align(f, np.array([[2.0, 3.0, 14.0, 17.0]]), 7, 1.0, 2), 3.25, rtol=1e-14)
    ramp = np.broadcast_to(np.arange(W, dtype=float), (C, H, W))
    x1, x2 = 2.0, 16.0
    out = ops.roi_align(ramp, np.array([[x1, 1.0, x2, 9.0]]), 7, 1.0, 2)
    bw = (x2 - x1) / 7
    expect = [x1 + pw * bw + 0.5 * bw for pw in range(7)]                    # mean of (i+0.5)/2 offsets
    np.testing.assert_allclose(out[0, 0, 0], expect, rtol=1e-12)


def test_roi_levels_vs_torchvision_level_mapper():
    from torchvision.ops.poolers import LevelMapper
    g = np.random.default_rng(5)
    xy = g.uniform(0, 500, (400, 2))
    rois = np.concatenate([xy, xy + g.uniform(0, 700, (400, 2))], axis=1)
    rois[0] = 0
    ref = LevelMapper(2, 5)([torch.from_numpy(rois)]).numpy()
    np.testing.assert_array_equal(ops.roi_levels(rois, 2, 5, (224, 4)), ref)


def test_rpn_merge_and_level_special_cases():
    """rpn_level with every anchor identical in score keeps index order and NMS keeps
    one box per duplicate cluster; rpn_merge pads with zero rows."""
    cls = np.zeros((1, 3, 2, 2))
    box = np.zeros((1, 12, 2, 2))
    out = ops.rpn_level(cls, box, 32, (0.5, 1.0, 2.0), 5, 0.7, 1e-3, (64, 64)).reshape(5, 6)
    anchors = ops.clip_boxes(ops.rpn_anchors(32, (0.5, 1.0, 2.0), (2, 2), (64, 64)), (64, 64))
    np.testing.assert_array_equal(out[:, :4], anchors[:5])                   # ties: lower index first
    merged = ops.rpn_merge([out.reshape(1, -1)], 8).reshape(8, 5)
    k = int(out[:, 5].sum())
    assert merged[:, 4].sum() == k and np.all(merged[k:] == 0)
