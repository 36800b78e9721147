"""Pins for oracle/model.py and the zoo: whole-model forward against torchvision
(fp64, CPU -- an independent implementation) and published parameter counts."""
import numpy as np
import pytest
import torch
import torchvision

from oracle import merge, model, ops
from workloads import synth, zoo

TV = {"resnet18": torchvision.models.resnet18, "resnet34": torchvision.models.resnet34,
      "resnet50": torchvision.models.resnet50, "resnet101": torchvision.models.resnet101,
      "resnet152": torchvision.models.resnet152, "vgg11": torchvision.models.vgg11,
      "vgg13": torchvision.models.vgg13, "vgg16": torchvision.models.vgg16,
      "vgg19": torchvision.models.vgg19, "alexnet": torchvision.models.alexnet}

# torchvision parameter counts (weights + biases + BN affine), SURVEY.md Appendix A.
PUBLISHED_PARAMS = {"resnet18": 11_689_512, "resnet34": 21_797_672, "resnet50": 25_557_032,
                    "resnet101": 44_549_160, "resnet152": 60_192_808, "vgg16": 138_357_544,
                    "vgg19": 143_667_240}


def _tv_param_count(layers):
    n = 0
    for l in layers:
        if l["op"] == "bn":
            n += 2 * l["c"]           # affine gamma/beta are parameters, running stats are buffers
        else:
            n += merge.param_count(l)
    return n


@pytest.mark.parametrize("name", sorted(PUBLISHED_PARAMS))
def test_param_counts_published(name):
    assert _tv_param_count(zoo.build(name)) == PUBLISHED_PARAMS[name]


@pytest.mark.parametrize("name", sorted(TV))
def test_param_counts_vs_torchvision(name):
    tv = TV[name](weights=None)
    assert _tv_param_count(zoo.build(name)) == sum(p.numel() for p in tv.parameters())


def _load_into_torchvision(name, layers, params):
    net = TV[name](weights=None).double().eval()
    mods = [m for m in net.modules() if isinstance(m, (torch.nn.Conv2d, torch.nn.BatchNorm2d, torch.nn.Linear))]
    ours = [(l, p) for l, p in zip(layers, params) if l["op"] in merge.PARAM_OPS]
    assert len(mods) == len(ours)
    with torch.no_grad():
        for m, (l, p) in zip(mods, ours):
            if l["op"] == "bn":
                assert isinstance(m, torch.nn.BatchNorm2d) and m.num_features == l["c"]
                m.weight.copy_(torch.from_numpy(p["gamma"].astype(np.float64)))
                m.bias.copy_(torch.from_numpy(p["beta"].astype(np.float64)))
                m.running_mean.copy_(torch.from_numpy(p["mean"].astype(np.float64)))
                m.running_var.copy_(torch.from_numpy(p["var"].astype(np.float64)))
            else:
                assert tuple(m.weight.shape) == p["w"].shape
                m.weight.copy_(torch.from_numpy(p["w"].astype(np.float64)))
                if "b" in p:
                    m.bias.copy_(torch.from_numpy(p["b"].astype(np.float64)))
                else:
                    assert m.bias is None
    return net


@pytest.mark.parametrize("name,res", [("resnet18", 64), ("resnet34", 64), ("resnet50", 64),
                                      ("vgg16", 32), ("alexnet", 96)])
def test_forward_matches_torchvision(name, res):
    layers = zoo.build(name)
    params = synth.params(layers, 99, 1)
    fr = synth.frames(99, 0, 2, res, res)
    ours = model.run(layers, params, fr)[-1]
    net = _load_into_torchvision(name, layers, params)
    with torch.no_grad():
        ref = net(torch.from_numpy(ops.preprocess(fr))).numpy()
    np.testing.assert_allclose(ours, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())


def test_shapes_resnet50_224():
    sh = model.shapes(zoo.build("resnet50"), (224, 224))
    assert sh[0] == (64, 112, 112)
    assert sh[3] == (64, 56, 56)
    assert sh[-1] == (1000,)
    assert sh[-3] == (2048, 1, 1)


def test_bf16_emulation_close_to_fp64():
    layers = zoo.build("resnet18")
    params = synth.params(layers, 5, 0)
    fr = synth.frames(5, 0, 1, 64, 64)
    a = model.run(layers, params, fr)[-1]
    b = model.run(layers, params, fr, emulate_bf16=True)[-1]
    rel = np.abs(a - b).max() / np.abs(a).max()
    assert 0 < rel < 0.05


def test_round_bf16_values():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 1e-40, 3.0e38])
    r = model.round_bf16(x)
    assert r[0] == 1.0
    assert r[1] == 1.0                      # tie -> even
    assert r[2] == 1.0 + 4 * 2 ** -8        # tie -> even (up)
    assert r[3] == -2.5
    # agrees with torch's bf16 conversion (RNE)
    t = torch.tensor(np.random.default_rng(0).standard_normal(1000), dtype=torch.float32)
    np.testing.assert_array_equal(model.round_bf16(t.numpy().astype(np.float64)),
                                  t.to(torch.bfloat16).to(torch.float64).numpy())


def test_storage_points_resnet_basic_block():
    layers = zoo.build("resnet18")
    st = model.storage_points(layers)
    # stem: conv(0) bn(1) relu(2) maxpool(3): only relu and pool materialised
    assert st[:4] == [False, False, True, True]
    # first basic block: conv bn relu conv bn add relu
    assert st[4:11] == [False, False, True, False, False, False, True]


def test_activations_stay_bounded_deep_resnet():
    """Input recipe check: random-init ResNet-152 keeps O(1)-O(100) activations."""
    layers = zoo.build("resnet152")
    params = synth.params(layers, 3, 0)
    vals = model.run(layers, params, synth.frames(3, 0, 1, 64, 64))
    mx = max(float(np.abs(v).max()) for v in vals)
    assert mx < 1e3
    assert float(np.abs(vals[-1]).std()) > 1e-2


# ----------------------------------------------------------------------------
# YOLOv3 / Tiny-YOLOv3 (darknet cfgs): published figures pin the zoo encoding,
# a torch interpreter of the same layer list pins the oracle's forward.
# ----------------------------------------------------------------------------

# darknet: yolov3.cfg 61,949,149 params / 140.69 BFLOPs @608 (65.86 @416);
# yolov3-tiny.cfg 8,852,366 params / 5.56 BFLOPs @416
DARKNET = {"yolov3": (61_949_149, 147, 75, {608: 140.69, 416: 65.86}),
           "tiny_yolov3": (8_852_366, 24, 13, {416: 5.56})}


def _conv_gflops(layers, res):
    sh = model.shapes(layers, (res, res))
    return sum(2 * s[0] * s[1] * s[2] * l["cin"] * l["k"][0] * l["k"][1]
               for l, s in zip(layers, sh) if l["op"] == "conv") / 1e9


@pytest.mark.parametrize("name", sorted(DARKNET))
def test_darknet_published_figures(name):
    params, n_param_layers, n_conv, gflops = DARKNET[name]
    layers = zoo.build(name)
    assert _tv_param_count(layers) == params
    assert sum(l["op"] in merge.PARAM_OPS for l in layers) == n_param_layers
    assert sum(l["op"] == "conv" for l in layers) == n_conv
    for res, g in gflops.items():
        assert round(_conv_gflops(layers, res), 2) == g


def test_yolov3_output_size():
    # 3 anchors x (19^2 + 38^2 + 76^2) cells = 22,743 boxes of 85 fields at 608
    sh = model.shapes(zoo.build("yolov3"), (608, 608))
    assert sh[-4] == (22_743 * 85,)          # the detection row (all decoded candidates)
    assert sh[-3] == (22_743 * 6,)           # candidates (x1, y1, x2, y2, score, label)
    assert sh[-2] == (1024 * 7,)             # the 1024 best: index + 6 fields
    assert sh[-1] == (100 * 6,)              # final detections after NMS (N2)


def test_yolo_decode_closed_form():
    """t = 0: centre = (cell + 0.5) * stride, size = anchor, scores = 0.5; t2 = ln 2 doubles w."""
    anchors, classes, h, w = ((10, 13), (16, 30)), 3, 2, 3
    x = np.zeros((1, 2 * 8, h, w))
    x[0, 8 + 2, 1, 2] = np.log(2.0)           # anchor 1, cell (1, 2): tw = ln 2
    x[0, 0, 0, 0] = 50.0                      # anchor 0, cell (0, 0): sigmoid(tx) -> 1
    y = ops.yolo_decode(x, anchors, classes, (64, 96)).reshape(1, 2, h, w, 8)
    sw, sh = 96 / w, 64 / h
    for a in range(2):
        for cy in range(h):
            for cx in range(w):
                box = y[0, a, cy, cx]
                exp_x = (1.0 + cx) * sw if (a, cy, cx) == (0, 0, 0) else (0.5 + cx) * sw
                assert box[0] == pytest.approx(exp_x, rel=1e-15, abs=1e-12)
                assert box[1] == pytest.approx((0.5 + cy) * sh)
                ew = anchors[a][0] * (2.0 if (a, cy, cx) == (1, 1, 2) else 1.0)
                assert box[2] == pytest.approx(ew) and box[3] == pytest.approx(anchors[a][1])
                np.testing.assert_allclose(box[4:], 0.5)


def _torch_forward(layers, params, frames_u8):
    """Independent fp64 interpreter of a layer list with torch.nn.functional ops."""
    import torch.nn.functional as F
    x0 = torch.from_numpy(ops.preprocess(frames_u8))
    vals = []
    for l, p in zip(layers, params):
        ins = [x0 if j < 0 else vals[j] for j in l["in"]]
        x, op = ins[0], l["op"]
        if op == "conv":
            b = torch.from_numpy(p["b"].astype(np.float64)) if "b" in p else None
            y = F.conv2d(x, torch.from_numpy(p["w"].astype(np.float64)), b, l["s"], l["p"], l["d"], l["groups"])
        elif op == "bn":
            y = F.batch_norm(x, *(torch.from_numpy(p[k].astype(np.float64)) for k in ("mean", "var", "gamma", "beta")),
                             training=False, eps=l["eps"])
        elif op == "leaky":
            y = F.leaky_relu(x, l["slope"])
        elif op == "relu":
            y = F.relu(x)
        elif op == "maxpool":
            if l.get("darknet"):
                kh, kw = l["k"]
                y = F.max_pool2d(F.pad(x, (0, kw - 1, 0, kh - 1), value=-np.inf), l["k"], l["s"])
            else:
                y = F.max_pool2d(x, l["k"], l["s"], l["p"], l["d"], ceil_mode=l["ceil"])
        elif op == "add":
            y = ins[0] + ins[1]
        elif op == "concat":
            y = torch.cat(ins, 1)
        elif op == "upsample":
            y = F.interpolate(x, scale_factor=l["scale"], mode="nearest")
        elif op == "yolo":
            n, _, h, w = x.shape
            A, nf = len(l["anchors"]), 5 + l["classes"]
            t = x.view(n, A, nf, h, w).permute(0, 1, 3, 4, 2)
            gy, gx = torch.meshgrid(torch.arange(h, dtype=torch.float64), torch.arange(w, dtype=torch.float64),
                                    indexing="ij")
            anc = torch.tensor(l["anchors"], dtype=torch.float64).view(1, A, 1, 1, 2)
            xy = (torch.sigmoid(t[..., :2]) + torch.stack([gx, gy], -1)) * torch.tensor(
                [x0.shape[3] / w, x0.shape[2] / h], dtype=torch.float64)
            y = torch.cat([xy, anc * torch.exp(t[..., 2:4]), torch.sigmoid(t[..., 4:])], -1).reshape(n, -1)
        elif op == "l2norm":
            y = F.normalize(x, dim=1) * torch.from_numpy(p["scale"].astype(np.float64)).view(1, -1, 1, 1)
        elif op == "ssd_decode":
            from torchvision.models.detection._utils import BoxCoder
            from torchvision.ops import boxes as box_ops
            loc, conf = ins
            n, _, h, w = loc.shape
            A, C = len(l["wh"]), l["classes"]
            ih, iw = x0.shape[2:]
            cx = ((torch.arange(w, dtype=torch.float64) + 0.5) * l["step"]).view(1, w, 1).expand(h, w, A)
            cy = ((torch.arange(h, dtype=torch.float64) + 0.5) * l["step"]).view(h, 1, 1).expand(h, w, A)
            aw = torch.tensor([q[0] for q in l["wh"]], dtype=torch.float64).view(1, 1, A).expand(h, w, A) * iw
            ah = torch.tensor([q[1] for q in l["wh"]], dtype=torch.float64).view(1, 1, A).expand(h, w, A) * ih
            anchors = torch.stack([cx - aw / 2, cy - ah / 2, cx + aw / 2, cy + ah / 2], -1).reshape(-1, 4)
            rel = loc.view(n, A, 4, h, w).permute(0, 3, 4, 1, 2).reshape(n, -1, 4)
            coder = BoxCoder(weights=l["weights"])
            boxes = torch.stack([box_ops.clip_boxes_to_image(coder.decode_single(rel[i], anchors), (ih, iw))
                                 for i in range(n)])
            prob = torch.softmax(conf.view(n, A, C, h, w).permute(0, 3, 4, 1, 2).reshape(n, -1, C), -1)
            y = torch.cat([boxes, prob[..., 1:].max(-1, keepdim=True).values, prob], -1).reshape(n, -1)
        elif op == "topk":
            rows = x.view(x.shape[0], -1, l["fields"])
            order = torch.sort(rows[..., l["score"]], dim=1, descending=True, stable=True).indices[:, :l["k"]]
            sel = torch.gather(rows, 1, order[..., None].expand(-1, -1, l["fields"]))
            y = torch.cat([order[..., None].to(torch.float64), sel], -1)
            pad = l["k"] - y.shape[1]                 # fewer candidates than k: index -1, zeros
            if pad > 0:
                fill = torch.zeros(y.shape[0], pad, y.shape[2], dtype=torch.float64)
                fill[..., 0] = -1
                y = torch.cat([y, fill], 1)
            y = y.reshape(x.shape[0], -1)
        elif op == "det_cand":
            r = x.view(x.shape[0], -1, l["fields"])
            if l["fmt"] == 1:
                best, lab = r[..., 5:].max(-1)
                box = torch.stack([r[..., 0] - r[..., 2] / 2, r[..., 1] - r[..., 3] / 2,
                                   r[..., 0] + r[..., 2] / 2, r[..., 1] + r[..., 3] / 2], -1)
                sc = r[..., 4] * best
            elif l["fmt"] == 2:
                best, lab = r[..., 6:].max(-1)
                box, sc, lab = r[..., :4], best, lab + 1
            else:
                box, sc, lab = r[..., :4], r[..., 4], r[..., 5].long()
            keep = (sc > l["score_thresh"]) & (box[..., 2] - box[..., 0] >= l["min_size"]) & \
                (box[..., 3] - box[..., 1] >= l["min_size"])
            y = torch.cat([box, torch.where(keep, sc, -1.0)[..., None], lab[..., None].to(torch.float64)], -1)
            y = y.reshape(x.shape[0], -1)
        elif op == "det_nms":
            import torchvision
            t = x.view(x.shape[0], -1, 7)
            y = torch.zeros(x.shape[0], l["max_det"], 6, dtype=torch.float64)
            y[..., 4] = -1
            for i in range(x.shape[0]):
                v = t[i][(t[i, :, 0] >= 0) & (t[i, :, 5] >= 0)]
                keep = torchvision.ops.batched_nms(v[:, 1:5], v[:, 5], v[:, 6].long(), l["iou"])[:l["max_det"]]
                y[i, :len(keep)] = v[keep][:, 1:]
            y = y.reshape(x.shape[0], -1)
        else:
            raise ValueError(op)
        vals.append(y)
    return vals[-1].numpy()


@pytest.mark.parametrize("name,res", [("tiny_yolov3", 64), ("yolov3", 64), ("ssd300", 300)])
def test_yolo_forward_matches_torch_interpreter(name, res):
    layers = zoo.build(name)
    params = synth.params(layers, 4, 0)
    frames = synth.frames(4, 0, 2, res, res)
    ours = model.run(layers, params, frames)[-1]
    ref = _torch_forward(layers, params, frames)
    assert ours.shape == ref.shape == (2, model.shapes(layers, (res, res))[-1][0])
    np.testing.assert_allclose(ours, ref, rtol=1e-9, atol=1e-9)


def test_storage_points_darknet_shortcut_and_heads():
    layers = zoo.build("tiny_yolov3")
    st = model.storage_points(layers)
    for i, l in enumerate(layers):
        if l["op"] == "yolo" or (i + 1 < len(layers) and layers[i + 1]["op"] == "yolo"):
            assert not st[i]                      # head output and decode: fp32
    y3 = zoo.build("yolov3")
    st3 = model.storage_points(y3)
    adds = [i for i, l in enumerate(y3) if l["op"] == "add"]
    assert all(st3[i] for i in adds)              # shortcut outputs are stored
    assert all(not st3[y3[i]["in"][0]] for i in adds)   # the fused leaky before each add is not


# ----------------------------------------------------------------------------
# SSD300-VGG16: torchvision's own DefaultBoxGenerator / BoxCoder / model pin the
# oracle's default boxes, decode and parameter count.
# ----------------------------------------------------------------------------

def test_ssd300_param_count_vs_torchvision():
    layers = zoo.build("ssd300")
    tv = torchvision.models.detection.ssd300_vgg16(weights=None, weights_backbone=None)
    n_tv = sum(p.numel() for p in tv.parameters())
    ours = sum(merge.param_count(l) for l in layers)
    assert ours == 35_641_314                      # SURVEY.md Appendix A (35 param layers)
    assert n_tv == ours + 512                      # + the L2Norm scale (not a param layer, R2)
    assert sum(l["op"] == "conv" for l in layers) == 35
    sh = model.shapes(layers, (300, 300))
    assert sh[-4] == (8732 * 96,)                  # 8732 default boxes x (4 + best + 91 classes)


def test_ssd_decode_vs_torchvision_boxcoder():
    from torchvision.models.detection.anchor_utils import DefaultBoxGenerator
    from torchvision.models.detection._utils import BoxCoder
    from torchvision.ops import boxes as box_ops
    from torchvision.models.detection.image_list import ImageList
    gen = DefaultBoxGenerator([[2], [2, 3], [2, 3], [2, 3], [2], [2]],
                              scales=[0.07, 0.15, 0.33, 0.51, 0.69, 0.87, 1.05], steps=[8, 16, 32, 64, 100, 300])
    sizes = [38, 19, 10, 5, 3, 1]
    feats = [torch.zeros(1, 1, s, s, dtype=torch.float64) for s in sizes]
    img = ImageList(torch.zeros(1, 3, 300, 300, dtype=torch.float64), [(300, 300)])
    anchors = gen(img, feats)[0]                   # [8732, 4] xyxy pixels
    coder = BoxCoder(weights=(10.0, 10.0, 5.0, 5.0))
    rng = np.random.default_rng(3)
    start = 0
    for k, s in enumerate(sizes):
        wh = zoo.ssd_wh_pairs(k)
        A, C = len(wh), 7
        loc = rng.standard_normal((1, A * 4, s, s)) * 2
        conf = rng.standard_normal((1, A * C, s, s))
        ours = ops.ssd_decode(loc, conf, wh, zoo._SSD_STEPS[k], C, (10.0, 10.0, 5.0, 5.0), (300, 300))
        ours = ours.reshape(-1, 5 + C)
        n = s * s * A
        rel = torch.from_numpy(loc.reshape(1, A, 4, s, s).transpose(0, 3, 4, 1, 2).reshape(-1, 4))
        ref = box_ops.clip_boxes_to_image(coder.decode_single(rel, anchors[start:start + n]), (300, 300))
        # torchvision keeps the default-box (w, h) pairs in float32: 1e-4 px absolute
        np.testing.assert_allclose(ours[:, :4], ref.numpy(), rtol=1e-6, atol=1e-4)
        logits = torch.from_numpy(conf.reshape(1, A, C, s, s).transpose(0, 3, 4, 1, 2).reshape(-1, C))
        p = torch.softmax(logits, -1).numpy()
        np.testing.assert_allclose(ours[:, 5:], p, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(ours[:, 4], p[:, 1:].max(-1), rtol=1e-12)
        start += n
    assert start == 8732


def test_l2norm_vs_torch():
    x = np.random.default_rng(1).standard_normal((2, 16, 3, 5))
    scale = np.linspace(1, 20, 16)
    ref = torch.nn.functional.normalize(torch.from_numpy(x), dim=1) * torch.from_numpy(scale).view(1, -1, 1, 1)
    np.testing.assert_allclose(ops.l2norm(x, scale, 1e-12), ref.numpy(), rtol=1e-13)
