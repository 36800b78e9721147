"""Model zoo: architectures of the paper's workloads as plain layer lists.

This module is *workload description* (input structure), shared by the oracle
and the CUDA path.  It holds none of the method's arithmetic: no signatures, no
grouping, no byte accounting, no shape inference, no convolution.  Each model
is an ordered list of layer dicts (a DAG in topological order); ``"in"`` lists
producer indices, ``-1`` is the model input (the preprocessed frame).

Layer dict keys (PyTorch constructor vocabulary, the paper's notion of a
layer's "type-specific properties"):

  conv    : cin, cout, k=(kh,kw), s=(sh,sw), p=(ph,pw), d=(dh,dw), groups, bias
  bn      : c, eps, momentum, affine, track
  relu    : -
  leaky   : slope
  maxpool : k, s, p, d, ceil   (+ "darknet": True for right/bottom-only pad)
  avgpool : k, s, p, ceil
  gap     : adaptive average pool to (oh, ow) = out
  add     : two inputs
  concat  : n inputs along channels (or along features for flat [N, F] inputs)
  upsample: scale (nearest)
  flatten : -
  linear  : fin, fout, bias
  yolo    : anchors ((w, h) pixels per anchor), classes -- YOLOv3 box decode
  l2norm  : c, eps -- x / max(||x||_channels, eps) * scale[c] (SSD conv4_3; scale is its param)
  ssd_decode: two inputs (loc head, conf head) of one feature map; wh ((w, h) per anchor,
            relative to the image), step, classes, weights -- SSD box decode (torchvision
            DefaultBoxGenerator + BoxCoder(10, 10, 5, 5), clipped) and class softmax
  topk    : k, fields, score -- per frame the k rows (of `fields` values) with the
            highest value in column `score`, ties by lower row index (the detectors'
            output step: top-100 candidates by objectness)
  rpn_level: two inputs (objectness head [A ch], box-delta head [4A ch]) of one FPN level;
            size, ratios (anchor generator), pre_n, nms, min_size -- Faster R-CNN RPN
            proposals of one level (anchors, BoxCoder(1,1,1,1) decode, top pre_n by
            objectness, clip, small-box removal, NMS)
  rpn_merge: the levels' rpn_level outputs; post_n -- the post_n highest-scoring kept
            proposals of a frame across levels
  roi_align: inputs (proposals, feature maps finest first); out, sampling, canonical
            (scale, level) -- MultiScaleRoIAlign; one [C, out, out] output per proposal
  box_post: inputs (class logits, box deltas, proposals); classes, weights -- Fast R-CNN
            box decode (BoxCoder(10, 10, 5, 5)) + softmax, one row per (proposal, class)
  det_cand: fmt (0 Fast R-CNN rows, 1 YOLO rows, 2 SSD rows), fields, score_thresh,
            min_size -- final detection candidates (x1, y1, x2, y2, score, label)
  det_nms : iou, max_det -- greedy batched NMS over a topk of det_cand rows (the final
            detections)

A conv may carry ``tie = j``: it applies layer j's parameters (the Faster R-CNN RPN
head is one set of weights run on every FPN level).  A tied conv is not a separate
layer: it has no parameters of its own and never appears in a shareable group.

Architectures follow torchvision 0.26 definitions (ResNet v1.5, VGG without BN,
AlexNet) -- the models the paper names in Table 1 and in its
overlap figures.
"""
from __future__ import annotations

import copy


class _B:
    """Tiny builder: appends layer dicts and returns their indices."""

    def __init__(self):
        self.layers = []

    def add(self, op, inp, **hp):
        d = {"op": op, "in": list(inp) if isinstance(inp, (list, tuple)) else [inp]}
        d.update(hp)
        self.layers.append(d)
        return len(self.layers) - 1

    def conv(self, x, cin, cout, k, s=1, p=0, d=1, bias=True, groups=1, tie=None):
        k = (k, k) if isinstance(k, int) else tuple(k)
        s = (s, s) if isinstance(s, int) else tuple(s)
        p = (p, p) if isinstance(p, int) else tuple(p)
        d = (d, d) if isinstance(d, int) else tuple(d)
        hp = {} if tie is None else {"tie": tie}
        return self.add("conv", x, cin=cin, cout=cout, k=k, s=s, p=p, d=d,
                        groups=groups, bias=bool(bias), **hp)

    def bn(self, x, c, eps=1e-5, momentum=0.1):
        return self.add("bn", x, c=c, eps=eps, momentum=momentum, affine=True, track=True)

    def relu(self, x):
        return self.add("relu", x)

    def leaky(self, x, slope=0.1):
        return self.add("leaky", x, slope=slope)

    def maxpool(self, x, k, s, p=0, ceil=False, darknet=False):
        return self.add("maxpool", x, k=(k, k), s=(s, s), p=(p, p), d=(1, 1),
                        ceil=bool(ceil), darknet=bool(darknet))

    def gap(self, x, out=(1, 1)):
        return self.add("gap", x, out=tuple(out))

    def addop(self, a, b):
        return self.add("add", [a, b])

    def concat(self, xs):
        return self.add("concat", list(xs))

    def upsample(self, x, scale=2):
        return self.add("upsample", x, scale=scale)

    def flatten(self, x):
        return self.add("flatten", x)

    def linear(self, x, fin, fout, bias=True):
        return self.add("linear", x, fin=fin, fout=fout, bias=bool(bias))

    def yolo(self, x, anchors, classes):
        return self.add("yolo", x, anchors=tuple(tuple(a) for a in anchors), classes=classes)

    def topk(self, x, k, fields, score):
        return self.add("topk", x, k=k, fields=fields, score=score)

    def det_cand(self, x, fmt, fields, score_thresh, min_size=0.0):
        return self.add("det_cand", x, fmt=fmt, fields=fields, score_thresh=float(score_thresh),
                        min_size=float(min_size))

    def det_nms(self, x, iou, max_det):
        return self.add("det_nms", x, iou=float(iou), max_det=max_det)

    def detect_tail(self, det, fmt, fields, score_thresh, min_size, iou, max_det, pre_n=1024):
        """Final detections: candidates -> the pre_n best by score -> greedy batched NMS."""
        cand = self.det_cand(det, fmt, fields, score_thresh, min_size)
        return self.det_nms(self.topk(cand, pre_n, 6, 4), iou, max_det)

    def l2norm(self, x, c, eps=1e-12):
        return self.add("l2norm", x, c=c, eps=eps)

    def rpn_level(self, cls, box, size, ratios, pre_n=1000, nms=0.7, min_size=1e-3):
        return self.add("rpn_level", [cls, box], size=size, ratios=tuple(ratios), pre_n=pre_n, nms=nms,
                        min_size=min_size)

    def rpn_merge(self, levels, post_n=1000):
        return self.add("rpn_merge", list(levels), post_n=post_n)

    def roi_align(self, props, feats, out=7, sampling=2, canonical=(224, 4)):
        return self.add("roi_align", [props] + list(feats), out=out, sampling=sampling,
                        canonical=tuple(canonical))

    def box_post(self, cls, box, props, classes, weights=(10.0, 10.0, 5.0, 5.0)):
        return self.add("box_post", [cls, box, props], classes=classes, weights=tuple(weights))

    def ssd_decode(self, loc, conf, wh, step, classes, weights=(10.0, 10.0, 5.0, 5.0)):
        return self.add("ssd_decode", [loc, conf], wh=tuple(tuple(p) for p in wh), step=step,
                        classes=classes, weights=tuple(weights))


# ----------------------------------------------------------------------------
# cfg1 tiny models: "2 tiny 4-layer CNNs sharing first 2 conv
# layers" (BASELINE.json configs[0]).  4 param layers each.
# ----------------------------------------------------------------------------

def tiny_a(num_classes=10):
    b = _B()
    x = b.conv(-1, 3, 16, 3, 1, 1)        # 0
    x = b.relu(x)                          # 1
    x = b.conv(x, 16, 32, 3, 2, 1)         # 2
    x = b.relu(x)                          # 3
    x = b.conv(x, 32, 32, 3, 2, 1)         # 4
    x = b.relu(x)                          # 5
    x = b.flatten(x)                       # 6
    b.linear(x, 32 * 8 * 8, num_classes)   # 7  (32x32 input -> 8x8)
    return b.layers


def tiny_b(num_classes=5):
    b = _B()
    x = b.conv(-1, 3, 16, 3, 1, 1)
    x = b.relu(x)
    x = b.conv(x, 16, 32, 3, 2, 1)
    x = b.relu(x)
    x = b.conv(x, 32, 64, 3, 2, 1)
    x = b.relu(x)
    x = b.flatten(x)
    b.linear(x, 64 * 8 * 8, num_classes)
    return b.layers


# ----------------------------------------------------------------------------
# ResNet (torchvision v1.5: stride on the 3x3 of the bottleneck)
# ----------------------------------------------------------------------------

def _basic(b, x, cin, cout, stride):
    idn = x
    y = b.conv(x, cin, cout, 3, stride, 1, bias=False)
    y = b.bn(y, cout)
    y = b.relu(y)
    y = b.conv(y, cout, cout, 3, 1, 1, bias=False)
    y = b.bn(y, cout)
    if stride != 1 or cin != cout:
        idn = b.conv(x, cin, cout, 1, stride, 0, bias=False)
        idn = b.bn(idn, cout)
    y = b.addop(y, idn)
    return b.relu(y), cout


def _bottleneck(b, x, cin, planes, stride):
    cout = planes * 4
    idn = x
    y = b.conv(x, cin, planes, 1, 1, 0, bias=False)
    y = b.bn(y, planes)
    y = b.relu(y)
    y = b.conv(y, planes, planes, 3, stride, 1, bias=False)
    y = b.bn(y, planes)
    y = b.relu(y)
    y = b.conv(y, planes, cout, 1, 1, 0, bias=False)
    y = b.bn(y, cout)
    if stride != 1 or cin != cout:
        idn = b.conv(x, cin, cout, 1, stride, 0, bias=False)
        idn = b.bn(idn, cout)
    y = b.addop(y, idn)
    return b.relu(y), cout


_RESNET = {18: ("basic", [2, 2, 2, 2]), 34: ("basic", [3, 4, 6, 3]),
           50: ("bottle", [3, 4, 6, 3]), 101: ("bottle", [3, 4, 23, 3]),
           152: ("bottle", [3, 8, 36, 3])}


def resnet(depth, num_classes=1000):
    kind, blocks = _RESNET[depth]
    b = _B()
    x = b.conv(-1, 3, 64, 7, 2, 3, bias=False)
    x = b.bn(x, 64)
    x = b.relu(x)
    x = b.maxpool(x, 3, 2, 1)
    c = 64
    for stage, (planes, n) in enumerate(zip([64, 128, 256, 512], blocks)):
        for i in range(n):
            stride = 2 if (stage > 0 and i == 0) else 1
            if kind == "basic":
                x, c = _basic(b, x, c, planes, stride)
            else:
                x, c = _bottleneck(b, x, c, planes, stride)
    x = b.gap(x, (1, 1))
    x = b.flatten(x)
    b.linear(x, c, num_classes)
    return b.layers


# ----------------------------------------------------------------------------
# VGG (torchvision, no BN) and AlexNet (for the VGG16/AlexNet overlap pin)
# ----------------------------------------------------------------------------

_VGG = {11: [64, "M", 128, "M", 256, 256, "M", 512, 512, "M", 512, 512, "M"],
        13: [64, 64, "M", 128, 128, "M", 256, 256, "M", 512, 512, "M", 512, 512, "M"],
        16: [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M",
             512, 512, 512, "M"],
        19: [64, 64, "M", 128, 128, "M", 256, 256, 256, 256, "M", 512, 512, 512, 512,
             "M", 512, 512, 512, 512, "M"]}


def vgg(depth, num_classes=1000):
    b = _B()
    x, c = -1, 3
    for v in _VGG[depth]:
        if v == "M":
            x = b.maxpool(x, 2, 2, 0)
        else:
            x = b.conv(x, c, v, 3, 1, 1)
            x = b.relu(x)
            c = v
    x = b.gap(x, (7, 7))
    x = b.flatten(x)
    x = b.linear(x, 512 * 7 * 7, 4096)
    x = b.relu(x)
    x = b.linear(x, 4096, 4096)
    x = b.relu(x)
    b.linear(x, 4096, num_classes)
    return b.layers


def alexnet(num_classes=1000):
    b = _B()
    x = b.conv(-1, 3, 64, 11, 4, 2)
    x = b.relu(x)
    x = b.maxpool(x, 3, 2)
    x = b.conv(x, 64, 192, 5, 1, 2)
    x = b.relu(x)
    x = b.maxpool(x, 3, 2)
    x = b.conv(x, 192, 384, 3, 1, 1)
    x = b.relu(x)
    x = b.conv(x, 384, 256, 3, 1, 1)
    x = b.relu(x)
    x = b.conv(x, 256, 256, 3, 1, 1)
    x = b.relu(x)
    x = b.maxpool(x, 3, 2)
    x = b.gap(x, (6, 6))
    x = b.flatten(x)
    x = b.linear(x, 256 * 6 * 6, 4096)
    x = b.relu(x)
    x = b.linear(x, 4096, 4096)
    x = b.relu(x)
    b.linear(x, 4096, num_classes)
    return b.layers


# ----------------------------------------------------------------------------
# YOLOv3 / Tiny-YOLOv3 (darknet cfgs yolov3.cfg, yolov3-tiny.cfg; 80 COCO
# classes): the detector family of the paper's workloads (SURVEY.md
# §8 cfg4/cfg5).  Darknet conv = conv(no bias) + BN + LeakyReLU(0.1); head convs
# are 1x1 with bias and linear activation; shortcut = branch + block input (no
# activation after the add); route = channel concat; upsample = nearest x2.
# ----------------------------------------------------------------------------

_COCO_ANCHORS = ((10, 13), (16, 30), (33, 23), (30, 61), (62, 45), (59, 119), (116, 90), (156, 198), (373, 326))
_TINY_ANCHORS = ((10, 14), (23, 27), (37, 58), (81, 82), (135, 169), (344, 319))


def _dconv(b, x, cin, cout, k, s=1):
    x = b.conv(x, cin, cout, k, s, (k - 1) // 2, bias=False)
    x = b.bn(x, cout)
    return b.leaky(x, 0.1)


def _head_conv(b, x, cin, classes):
    return b.conv(x, cin, 3 * (5 + classes), 1, 1, 0, bias=True)


def yolov3(classes=80):
    b = _B()
    x = _dconv(b, -1, 3, 32, 3)
    c = 32
    routes = []
    for cout, n in ((64, 1), (128, 2), (256, 8), (512, 8), (1024, 4)):
        x = _dconv(b, x, c, cout, 3, 2)
        c = cout
        for _ in range(n):
            y = _dconv(b, x, c, c // 2, 1)
            y = _dconv(b, y, c // 2, c, 3)
            x = b.addop(y, x)          # shortcut from=-3, linear
        routes.append(x)
    r36, r61 = routes[2], routes[3]
    outs = []
    # scale 1 (stride 32)
    y = x
    cin = 1024
    for i in range(5):
        y = _dconv(b, y, cin, 512 if i % 2 == 0 else 1024, 1 if i % 2 == 0 else 3)
        cin = 512 if i % 2 == 0 else 1024
    branch = y
    y = _dconv(b, y, 512, 1024, 3)
    outs.append(b.yolo(_head_conv(b, y, 1024, classes), _COCO_ANCHORS[6:9], classes))
    # scale 2 (stride 16)
    y = _dconv(b, branch, 512, 256, 1)
    y = b.concat([b.upsample(y, 2), r61])
    cin = 768
    for i in range(5):
        y = _dconv(b, y, cin, 256 if i % 2 == 0 else 512, 1 if i % 2 == 0 else 3)
        cin = 256 if i % 2 == 0 else 512
    branch = y
    y = _dconv(b, y, 256, 512, 3)
    outs.append(b.yolo(_head_conv(b, y, 512, classes), _COCO_ANCHORS[3:6], classes))
    # scale 3 (stride 8)
    y = _dconv(b, branch, 256, 128, 1)
    y = b.concat([b.upsample(y, 2), r36])
    cin = 384
    for i in range(5):
        y = _dconv(b, y, cin, 128 if i % 2 == 0 else 256, 1 if i % 2 == 0 else 3)
        cin = 128 if i % 2 == 0 else 256
    y = _dconv(b, y, 128, 256, 3)
    outs.append(b.yolo(_head_conv(b, y, 256, classes), _COCO_ANCHORS[0:3], classes))
    det = b.concat(outs)               # all decoded boxes, [N, boxes * (5 + classes)]
    # final detections: conf = obj * best class > 0.25, IoU 0.45, 100 per frame (R22)
    b.detect_tail(det, 1, 5 + classes, 0.25, 0.0, 0.45, 100)
    return b.layers


def tiny_yolov3(classes=80):
    b = _B()
    x = _dconv(b, -1, 3, 16, 3)
    x = b.maxpool(x, 2, 2)
    c = 16
    route = None
    for cout in (32, 64, 128, 256):
        x = _dconv(b, x, c, cout, 3)
        c = cout
        if cout == 256:
            route = x
        x = b.maxpool(x, 2, 2)
    x = _dconv(b, x, 256, 512, 3)
    x = b.maxpool(x, 2, 1, darknet=True)   # 2x2 stride 1, right/bottom pad (13 -> 13)
    x = _dconv(b, x, 512, 1024, 3)
    branch = _dconv(b, x, 1024, 256, 1)
    y = _dconv(b, branch, 256, 512, 3)
    o1 = b.yolo(_head_conv(b, y, 512, classes), _TINY_ANCHORS[3:6], classes)
    y = _dconv(b, branch, 256, 128, 1)
    y = b.concat([b.upsample(y, 2), route])
    y = _dconv(b, y, 384, 256, 3)
    o2 = b.yolo(_head_conv(b, y, 256, classes), _TINY_ANCHORS[1:4], classes)
    det = b.concat([o1, o2])
    b.detect_tail(det, 1, 5 + classes, 0.25, 0.0, 0.45, 100)
    return b.layers


# ----------------------------------------------------------------------------
# SSD300-VGG16 (torchvision ssd300_vgg16, 91 COCO classes): VGG16 base with
# ceil-mode pool3, L2-normalised conv4_3, pool5 3x3/s1, dilated conv6 + conv7,
# four extra blocks, 3x3 loc/conf heads on 6 maps (38, 19, 10, 5, 3, 1), 8732
# default boxes.  Output: top-100 decoded boxes by best foreground probability.
# ----------------------------------------------------------------------------

_SSD_AR = ((2,), (2, 3), (2, 3), (2, 3), (2,), (2,))
_SSD_SCALES = (0.07, 0.15, 0.33, 0.51, 0.69, 0.87, 1.05)
_SSD_STEPS = (8, 16, 32, 64, 100, 300)


def ssd_wh_pairs(k):
    """Default-box (w, h) pairs of map k relative to the image (DefaultBoxGenerator,
    clip=True): (s_k, s_k), (s', s') with s' = sqrt(s_k s_k+1), then per aspect
    ratio r: (s_k sqrt r, s_k / sqrt r), (s_k / sqrt r, s_k sqrt r)."""
    import math
    s, s2 = _SSD_SCALES[k], math.sqrt(_SSD_SCALES[k] * _SSD_SCALES[k + 1])
    pairs = [(s, s), (s2, s2)]
    for r in _SSD_AR[k]:
        q = math.sqrt(r)
        pairs += [(s * q, s / q), (s / q, s * q)]
    return tuple((min(max(w, 0.0), 1.0), min(max(h, 0.0), 1.0)) for w, h in pairs)


def ssd300(classes=91):
    b = _B()
    x, c = -1, 3
    for v in (64, 64, "M", 128, 128, "M", 256, 256, 256, "C", 512, 512, 512):
        if v == "M":
            x = b.maxpool(x, 2, 2)
        elif v == "C":
            x = b.maxpool(x, 2, 2, ceil=True)
        else:
            x = b.relu(b.conv(x, c, v, 3, 1, 1))
            c = v
    feats = [(b.l2norm(x, 512), 512)]
    x = b.maxpool(x, 2, 2)
    for _ in range(3):
        x = b.relu(b.conv(x, 512, 512, 3, 1, 1))
    x = b.maxpool(x, 3, 1, 1)
    x = b.relu(b.conv(x, 512, 1024, 3, 1, 6, d=6))
    x = b.relu(b.conv(x, 1024, 1024, 1))
    feats.append((x, 1024))
    for cin, mid, cout, s, p in ((1024, 256, 512, 2, 1), (512, 128, 256, 2, 1), (256, 128, 256, 1, 0),
                                 (256, 128, 256, 1, 0)):
        x = b.relu(b.conv(x, cin, mid, 1))
        x = b.relu(b.conv(x, mid, cout, 3, s, p))
        feats.append((x, cout))
    decs = []
    for k, (f, cf) in enumerate(feats):
        wh = ssd_wh_pairs(k)
        loc = b.conv(f, cf, len(wh) * 4, 3, 1, 1)
        conf = b.conv(f, cf, len(wh) * classes, 3, 1, 1)
        decs.append(b.ssd_decode(loc, conf, wh, _SSD_STEPS[k], classes))
    det = b.concat(decs)                        # [N, 8732 * (5 + classes)]
    # torchvision SSD: score > 0.01, NMS 0.45, 200 detections per frame (R22)
    b.detect_tail(det, 2, 5 + classes, 0.01, 0.0, 0.45, 200)
    return b.layers


# ----------------------------------------------------------------------------
# Faster R-CNN ResNet-50-FPN (torchvision fasterrcnn_resnet50_fpn, 91 COCO classes;
# SURVEY.md §8 cfg4).  ResNet-50 trunk (C2..C5), FPN (1x1 lateral + nearest x2
# top-down + 3x3 output convs, P6 = 1x1/s2 max pool), RPN head (3x3 conv + ReLU,
# 1x1 objectness and box-delta convs) -- ONE weight set applied to all five levels
# (tied), anchors 32..512 x ratios (0.5, 1, 2), 1000 proposals per level before and
# 1000 per frame after NMS(0.7); MultiScaleRoIAlign 7x7 (sampling 2) over P2..P5;
# TwoMLPHead (fc6, fc7) and the box predictor; output: the top-100 (proposal,
# class) candidates by class probability.  Frame sizes must be multiples of 32 (the
# torchvision transform pads to 32; its 800-pixel resize is not applied -- frames
# arrive at the configured resolution).  Param layers are built in torchvision's
# state_dict order (trunk, fpn.inner_blocks, fpn.layer_blocks, rpn.head, box head).
# ----------------------------------------------------------------------------

def frcnn_r50_fpn(classes=91):
    b = _B()
    x = b.conv(-1, 3, 64, 7, 2, 3, bias=False)
    x = b.relu(b.bn(x, 64))
    x = b.maxpool(x, 3, 2, 1)
    c, cs = 64, []
    for stage, (planes, n) in enumerate(zip([64, 128, 256, 512], [3, 4, 6, 3])):
        for i in range(n):
            x, c = _bottleneck(b, x, c, planes, 2 if (stage > 0 and i == 0) else 1)
        cs.append((x, c))
    inner = [b.conv(xc, cc, 256, 1) for xc, cc in cs]
    td = [None, None, None, inner[3]]
    for i in (2, 1, 0):
        td[i] = b.addop(inner[i], b.upsample(td[i + 1], 2))
    feats = [b.conv(t, 256, 256, 3, 1, 1) for t in td]
    feats.append(b.maxpool(feats[3], 1, 2, 0))           # LastLevelMaxPool (P6)
    levels, tied = [], None
    for lv, f in enumerate(feats):
        t = b.conv(f, 256, 256, 3, 1, 1, tie=None if tied is None else tied[0])
        h = b.relu(t)
        cl = b.conv(h, 256, 3, 1, tie=None if tied is None else tied[1])
        bb = b.conv(h, 256, 12, 1, tie=None if tied is None else tied[2])
        if tied is None:
            tied = (t, cl, bb)
        levels.append(b.rpn_level(cl, bb, 32 << lv, (0.5, 1.0, 2.0)))
    props = b.rpn_merge(levels, 1000)
    roi = b.roi_align(props, feats[:4], 7, 2)
    x = b.flatten(roi)
    x = b.relu(b.linear(x, 256 * 7 * 7, 1024))
    x = b.relu(b.linear(x, 1024, 1024))
    cls = b.linear(x, 1024, classes)
    box = b.linear(x, 1024, classes * 4)
    det = b.box_post(cls, box, props, classes)            # [N, 1000 * (classes-1) * 6]
    # torchvision RoIHeads: min size 1e-2, NMS 0.5, 100 per frame; score threshold 0.011
    # instead of 0.05 (random-init softmax is ~1/91 everywhere, reading R22)
    b.detect_tail(det, 0, 6, 0.011, 1e-2, 0.5, 100)
    return b.layers


MODELS = {
    "tiny_a": tiny_a, "tiny_b": tiny_b,
    "resnet18": lambda: resnet(18), "resnet34": lambda: resnet(34),
    "resnet50": lambda: resnet(50), "resnet101": lambda: resnet(101),
    "resnet152": lambda: resnet(152),
    "vgg11": lambda: vgg(11), "vgg13": lambda: vgg(13),
    "vgg16": lambda: vgg(16), "vgg19": lambda: vgg(19),
    "alexnet": alexnet,
    "yolov3": yolov3, "tiny_yolov3": tiny_yolov3, "ssd300": ssd300,
    "frcnn_r50_fpn": frcnn_r50_fpn,
}


def build(name):
    return copy.deepcopy(MODELS[name]())


PARAM_OPS = ("conv", "bn", "linear")
