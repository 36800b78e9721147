"""Oracle layer operators: NumPy fp64, NCHW, PyTorch eval-mode semantics.

Test infrastructure only (see oracle/__init__.py).  Each operator is the plain
definition of the layer type the paper's models are built from (PAPER.md:209-211:
"a layer type (e.g., convolutional, linear, batch normalization), which in turn
indicates how the layer transforms inputs").  Merging does not change what a
layer computes, only where its weights live, so these are the
unmerged definitions.
"""
from __future__ import annotations

import math

import numpy as np

IMAGENET_MEAN = np.array([0.485, 0.456, 0.406])
IMAGENET_STD = np.array([0.229, 0.224, 0.225])


def preprocess(frames_u8):
    """uint8 [N,H,W,3] -> fp64 NCHW, x = (u8/255 - mean)/std (ImageNet constants)."""
    x = frames_u8.astype(np.float64) / 255.0
    x = (x - IMAGENET_MEAN) / IMAGENET_STD
    return np.ascontiguousarray(x.transpose(0, 3, 1, 2))


def conv_out_size(h, k, s, p, d):
    return (h + 2 * p - d * (k - 1) - 1) // s + 1


def conv2d(x, w, b, s, p, d, groups=1):
    """Direct convolution: y[n,co,i,j] = b[co] + sum_{ci,r,t} w[co,ci,r,t] *
    xpad[n, ci, i*sh + r*dh, j*sw + t*dw]  (zero padding).

    Implemented as a sum over filter taps (r,t) of fp64 matmuls of the shifted,
    strided input window -- no im2col, Winograd or FFT.
    """
    n, cin, h, wd = x.shape
    cout, cin_g, kh, kw = w.shape
    sh, sw = s
    ph, pw = p
    dh, dw = d
    ho = conv_out_size(h, kh, sh, ph, dh)
    wo = conv_out_size(wd, kw, sw, pw, dw)
    xp = np.zeros((n, cin, h + 2 * ph, wd + 2 * pw), dtype=np.float64)
    xp[:, :, ph:ph + h, pw:pw + wd] = x
    y = np.zeros((n, cout, ho, wo), dtype=np.float64)
    cout_g = cout // groups
    for g in range(groups):
        ci0, co0 = g * cin_g, g * cout_g
        for r in range(kh):
            for t in range(kw):
                win = xp[:, ci0:ci0 + cin_g,
                         r * dh: r * dh + sh * (ho - 1) + 1: sh,
                         t * dw: t * dw + sw * (wo - 1) + 1: sw]          # [n, cin_g, ho, wo]
                wt = w[co0:co0 + cout_g, :, r, t].astype(np.float64)     # [cout_g, cin_g]
                y[:, co0:co0 + cout_g] += np.einsum("oc,nchw->nohw", wt, win, optimize=True)
    if b is not None:
        y += np.asarray(b, dtype=np.float64)[None, :, None, None]
    return y


def batchnorm(x, gamma, beta, mean, var, eps):
    """Eval-mode BN: gamma * (x - mean) / sqrt(var + eps) + beta, per channel."""
    sh = (1, -1) + (1,) * (x.ndim - 2)
    g = np.asarray(gamma, np.float64).reshape(sh)
    bt = np.asarray(beta, np.float64).reshape(sh)
    m = np.asarray(mean, np.float64).reshape(sh)
    v = np.asarray(var, np.float64).reshape(sh)
    return g * (x - m) / np.sqrt(v + eps) + bt


def relu(x):
    return np.maximum(x, 0.0)


def leaky_relu(x, slope):
    return np.where(x >= 0, x, x * slope)


def pool_out_size(h, k, s, p, d, ceil):
    num = h + 2 * p - d * (k - 1) - 1
    if ceil:
        o = -(-num // s) + 1
        if (o - 1) * s >= h + p:      # PyTorch: last window must start inside input or left pad
            o -= 1
    else:
        o = num // s + 1
    return o


def maxpool2d(x, k, s, p, d=(1, 1), ceil=False, darknet=False):
    """Max pool with -inf padding (PyTorch semantics, incl. ceil_mode).

    darknet=True: darknet's maxpool (pad size-1 on the right/bottom only, i.e.
    out-of-range taps ignored), the Tiny-YOLOv3 reading in DESIGN.md.
    """
    n, c, h, w = x.shape
    (kh, kw), (sh, sw), (ph, pw), (dh, dw) = k, s, p, d
    if darknet:
        ho, wo = (h - 1) // sh + 1, (w - 1) // sw + 1
        top, left = 0, 0
        hp, wp = h + kh - 1, w + kw - 1
    else:
        ho = pool_out_size(h, kh, sh, ph, dh, ceil)
        wo = pool_out_size(w, kw, sw, pw, dw, ceil)
        top, left = ph, pw
        hp = max(h + 2 * ph, (ho - 1) * sh + dh * (kh - 1) + 1)
        wp = max(w + 2 * pw, (wo - 1) * sw + dw * (kw - 1) + 1)
    xp = np.full((n, c, hp, wp), -np.inf, dtype=np.float64)
    xp[:, :, top:top + h, left:left + w] = x
    y = np.full((n, c, ho, wo), -np.inf, dtype=np.float64)
    for r in range(kh):
        for t in range(kw):
            win = xp[:, :, r * dh: r * dh + sh * (ho - 1) + 1: sh, t * dw: t * dw + sw * (wo - 1) + 1: sw]
            y = np.maximum(y, win)
    return y


def adaptive_avgpool2d(x, out):
    """PyTorch adaptive average pool: bin i spans [floor(i*H/oh), ceil((i+1)*H/oh))."""
    n, c, h, w = x.shape
    oh, ow = out
    y = np.zeros((n, c, oh, ow), dtype=np.float64)
    for i in range(oh):
        h0, h1 = (i * h) // oh, -(-((i + 1) * h) // oh)
        for j in range(ow):
            w0, w1 = (j * w) // ow, -(-((j + 1) * w) // ow)
            y[:, :, i, j] = x[:, :, h0:h1, w0:w1].mean(axis=(2, 3))
    return y


def add(a, b):
    return a + b


def concat(xs):
    return np.concatenate(xs, axis=1)


def upsample_nearest(x, scale):
    return x.repeat(scale, axis=2).repeat(scale, axis=3)


def flatten(x):
    """NCHW flatten (PyTorch order): [N, C*H*W] with W fastest."""
    return x.reshape(x.shape[0], -1)


def linear(x, w, b):
    y = x @ np.asarray(w, np.float64).T
    if b is not None:
        y = y + np.asarray(b, np.float64)
    return y


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def yolo_decode(x, anchors, classes, in_hw):
    """YOLOv3 box decode of one head (darknet yolo layer).

    x: head conv output [N, A*(5+classes), H, W] (NCHW).  For anchor a, cell
    (cy, cx) and the raw values t = x[n, a*(5+classes) + f, cy, cx]:
      bx = (sigmoid(t0) + cx) * stride_w,  by = (sigmoid(t1) + cy) * stride_h,
      bw = anchor_w * exp(t2),             bh = anchor_h * exp(t3),
      objectness = sigmoid(t4),            class k = sigmoid(t(5+k)),
    with stride = network input size / feature size.  Output [N, A*H*W*(5+classes)]
    in (a, cy, cx, field) order -- one row of 5+classes fields per candidate box.
    """
    n, ch, h, w = x.shape
    A, F = len(anchors), 5 + classes
    assert ch == A * F
    sw, sh = in_hw[1] / w, in_hw[0] / h
    t = x.reshape(n, A, F, h, w).transpose(0, 1, 3, 4, 2)     # [n, a, cy, cx, f]
    out = np.empty_like(t, dtype=np.float64)
    cx = np.arange(w, dtype=np.float64)[None, None, None, :]
    cy = np.arange(h, dtype=np.float64)[None, None, :, None]
    aw = np.array([a[0] for a in anchors], np.float64)[None, :, None, None]
    ah = np.array([a[1] for a in anchors], np.float64)[None, :, None, None]
    out[..., 0] = (sigmoid(t[..., 0]) + cx) * sw
    out[..., 1] = (sigmoid(t[..., 1]) + cy) * sh
    out[..., 2] = aw * np.exp(t[..., 2])
    out[..., 3] = ah * np.exp(t[..., 3])
    out[..., 4:] = sigmoid(t[..., 4:])
    return out.reshape(n, -1)


def l2norm(x, scale, eps):
    """SSD's L2Norm: x / max(||x||_2 over channels, eps) * scale[c] (torchvision
    F.normalize(x) * scale_weight)."""
    n = np.sqrt((x * x).sum(axis=1, keepdims=True))
    return x / np.maximum(n, eps) * np.asarray(scale, np.float64)[None, :, None, None]


def ssd_decode(loc, conf, wh, step, classes, weights, in_hw):
    """SSD box decode of one feature map (torchvision DefaultBoxGenerator(clip=True)
    + BoxCoder(weights).decode_single + clip_boxes_to_image) and class softmax.

    loc [N, A*4, H, W], conf [N, A*classes, H, W].  Default box of cell (cy, cx),
    anchor a: centre ((cx+0.5)*step, (cy+0.5)*step) in pixels (step = image / f
    factor as torchvision: image_size / step cells), size wh[a] * (img_w, img_h).
    With (dx, dy, dw, dh) = loc / weights, dw, dh <= log(1000/16):
      ctr = d * anchor_size + anchor_ctr, size = exp(d) * anchor_size,
      box = (ctr - size/2, ctr + size/2) clipped to the image.
    Rows in (cy, cx, a) order: x1, y1, x2, y2, best foreground probability
    (max over classes 1..), then the softmax over all classes.  [N, H*W*A*(5+classes)]
    """
    n, _, h, w = loc.shape
    A = len(wh)
    img_h, img_w = in_hw
    d = loc.reshape(n, A, 4, h, w).transpose(0, 3, 4, 1, 2)          # [n, cy, cx, a, 4]
    lg = conf.reshape(n, A, classes, h, w).transpose(0, 3, 4, 1, 2)  # [n, cy, cx, a, C]
    x_f, y_f = img_w / step, img_h / step
    acx = ((np.arange(w) + 0.5) / x_f)[None, :, None] * img_w
    acy = ((np.arange(h) + 0.5) / y_f)[:, None, None] * img_h
    aw = np.array([p[0] for p in wh])[None, None, :] * img_w
    ah = np.array([p[1] for p in wh])[None, None, :] * img_h
    # anchors as xyxy, then back to centre/size the way BoxCoder does
    x1, x2 = acx - 0.5 * aw, acx + 0.5 * aw
    y1, y2 = acy - 0.5 * ah, acy + 0.5 * ah
    widths, heights = x2 - x1, y2 - y1
    ctr_x, ctr_y = x1 + 0.5 * widths, y1 + 0.5 * heights
    clamp = np.log(1000.0 / 16)
    dx, dy = d[..., 0] / weights[0], d[..., 1] / weights[1]
    dw, dh = np.minimum(d[..., 2] / weights[2], clamp), np.minimum(d[..., 3] / weights[3], clamp)
    pcx, pcy = dx * widths + ctr_x, dy * heights + ctr_y
    pw, ph = np.exp(dw) * widths, np.exp(dh) * heights
    out = np.empty((n, h, w, A, 5 + classes))
    out[..., 0] = np.clip(pcx - 0.5 * pw, 0, img_w)
    out[..., 1] = np.clip(pcy - 0.5 * ph, 0, img_h)
    out[..., 2] = np.clip(pcx + 0.5 * pw, 0, img_w)
    out[..., 3] = np.clip(pcy + 0.5 * ph, 0, img_h)
    e = np.exp(lg - lg.max(axis=-1, keepdims=True))
    p = e / e.sum(axis=-1, keepdims=True)
    out[..., 5:] = p
    out[..., 4] = p[..., 1:].max(axis=-1)
    return out.reshape(n, -1)


def topk_rows(x, k, fields, score):
    """Top-k candidate rows per frame: x [N, n*fields] holds n
    rows of `fields` values; rows are ranked by x[row*fields + score] descending, ties
    by lower row index (a total order, so the selection is unique).  Output
    [N, k*(fields+1)]: per selected row its index (as a float) then its fields;
    rows beyond n are index -1 and zeros."""
    n_img = x.shape[0]
    n = x.shape[1] // fields
    rows = x.reshape(n_img, n, fields)
    out = np.zeros((n_img, k, fields + 1), dtype=np.float64)
    out[:, :, 0] = -1.0
    for i in range(n_img):
        order = np.lexsort((np.arange(n), -rows[i, :, score]))[:k]
        out[i, :len(order), 0] = order
        out[i, :len(order), 1:] = rows[i, order]
    return out.reshape(n_img, -1)


# ----------------------------------------------------------------------------
# Faster R-CNN (torchvision fasterrcnn_resnet50_fpn, eval mode; SURVEY.md §8(a)
# a9 "RPN top-k + NMS(0.7) + MultiScaleRoIAlign(7x7, sr = 2)", a8 large-M box head)
# ----------------------------------------------------------------------------

BBOX_XFORM_CLIP = math.log(1000.0 / 16)


def rpn_anchors(size, ratios, feat_hw, img_hw):
    """AnchorGenerator for one level: base anchors round([-w, -h, w, h] / 2) with
    h = size*sqrt(r), w = size/sqrt(r) (ratio-major), shifted by (x, y)*stride with
    stride = image // feature (integer division).  [H*W*A, 4] in (y, x, a) order."""
    base = []
    for r in ratios:
        hr = math.sqrt(r)
        wr = 1.0 / hr
        base.append(np.round(np.array([-wr * size, -hr * size, wr * size, hr * size]) / 2.0))
    base = np.array(base)                                        # [A, 4]
    fh, fw = feat_hw
    sy, sx = img_hw[0] // fh, img_hw[1] // fw
    ys, xs = np.meshgrid(np.arange(fh) * sy, np.arange(fw) * sx, indexing="ij")
    shifts = np.stack([xs.ravel(), ys.ravel(), xs.ravel(), ys.ravel()], axis=1).astype(np.float64)
    return (shifts[:, None, :] + base[None, :, :]).reshape(-1, 4)


def box_decode(deltas, boxes, weights):
    """torchvision BoxCoder.decode_single: deltas [..., 4] relative to boxes [..., 4]
    (x1, y1, x2, y2); dw, dh clamped at log(1000/16)."""
    wx, wy, ww, wh = weights
    widths = boxes[..., 2] - boxes[..., 0]
    heights = boxes[..., 3] - boxes[..., 1]
    ctr_x = boxes[..., 0] + 0.5 * widths
    ctr_y = boxes[..., 1] + 0.5 * heights
    dx, dy = deltas[..., 0] / wx, deltas[..., 1] / wy
    dw = np.minimum(deltas[..., 2] / ww, BBOX_XFORM_CLIP)
    dh = np.minimum(deltas[..., 3] / wh, BBOX_XFORM_CLIP)
    pcx, pcy = dx * widths + ctr_x, dy * heights + ctr_y
    pw, ph = np.exp(dw) * widths, np.exp(dh) * heights
    return np.stack([pcx - 0.5 * pw, pcy - 0.5 * ph, pcx + 0.5 * pw, pcy + 0.5 * ph], axis=-1)


def clip_boxes(boxes, img_hw):
    """clip_boxes_to_image: x into [0, W], y into [0, H]."""
    out = boxes.copy()
    out[..., 0::2] = np.clip(out[..., 0::2], 0, img_hw[1])
    out[..., 1::2] = np.clip(out[..., 1::2], 0, img_hw[0])
    return out


def nms(boxes, scores, thresh):
    """Greedy NMS (torchvision.ops.nms): visit boxes by score descending (ties by
    lower index, a stable sort), keep a box unless an already kept box overlaps it
    with IoU > thresh; IoU = inter / (area_i + area_j - inter).  Returns kept
    indices in visiting order."""
    order = np.lexsort((np.arange(len(scores)), -np.asarray(scores)))
    area = (boxes[:, 2] - boxes[:, 0]) * (boxes[:, 3] - boxes[:, 1])
    suppressed = np.zeros(len(scores), bool)
    keep = []
    for i in order:
        if suppressed[i]:
            continue
        keep.append(int(i))
        iw = np.maximum(0.0, np.minimum(boxes[i, 2], boxes[:, 2]) - np.maximum(boxes[i, 0], boxes[:, 0]))
        ih = np.maximum(0.0, np.minimum(boxes[i, 3], boxes[:, 3]) - np.maximum(boxes[i, 1], boxes[:, 1]))
        inter = iw * ih
        with np.errstate(invalid="ignore", divide="ignore"):
            iou = inter / (area[i] + area - inter)
        suppressed |= iou > thresh                          # NaN (0/0) never suppresses
    return keep


def rpn_level(cls, box, size, ratios, pre_n, nms_thresh, min_size, img_hw):
    """RPN proposals of one FPN level (torchvision RegionProposalNetwork, eval:
    decode -> _get_top_n_idx -> clip -> remove_small_boxes -> batched_nms, whose
    per-level NMS is this level's own).

    cls [N, A, H, W] objectness logits, box [N, 4A, H, W] deltas (channel a*4+j).
    Anchors (rpn_anchors) in (y, x, a) order; BoxCoder(1, 1, 1, 1) decode; the
    K = min(pre_n, H*W*A) anchors with the highest logit (ties by lower index,
    reading: torch.topk leaves ties unspecified), in that order; boxes clipped to
    the image; keep = width >= min_size and height >= min_size and not suppressed
    by NMS(nms_thresh) among the kept boxes of this level (sigmoid is monotonic,
    so ranking by probability = ranking by logit; score_thresh 0 keeps all).
    Output [N, K*6]: rows (x1, y1, x2, y2, logit, keep)."""
    n, A, h, w = cls.shape
    anchors = rpn_anchors(size, ratios, (h, w), img_hw)
    logit = cls.transpose(0, 2, 3, 1).reshape(n, -1)                   # (y, x, a)
    d = box.reshape(n, A, 4, h, w).transpose(0, 3, 4, 1, 2).reshape(n, -1, 4)
    K = min(pre_n, h * w * A)
    out = np.zeros((n, K, 6))
    for i in range(n):
        top = np.lexsort((np.arange(logit.shape[1]), -logit[i]))[:K]
        b = clip_boxes(box_decode(d[i, top], anchors[top], (1.0, 1.0, 1.0, 1.0)), img_hw)
        ok = ((b[:, 2] - b[:, 0]) >= min_size) & ((b[:, 3] - b[:, 1]) >= min_size)
        cand = np.nonzero(ok)[0]
        kept = cand[nms(b[cand], logit[i, top][cand], nms_thresh)]
        out[i, :, :4] = b
        out[i, :, 4] = logit[i, top]
        out[i, kept, 5] = 1.0
    return out.reshape(n, -1)


def rpn_merge(levels, post_n):
    """A frame's proposals: the kept rows of every level (rpn_level), ranked by score
    descending (ties by lower index in level-concatenated order), the first post_n
    (batched_nms's final sort, then keep[:post_n]).  Output [N, post_n*5]: rows
    (x1, y1, x2, y2, 1); missing rows (fewer kept boxes) are (0, 0, 0, 0, 0)."""
    rows = np.concatenate([lv.reshape(lv.shape[0], -1, 6) for lv in levels], axis=1)
    n = rows.shape[0]
    out = np.zeros((n, post_n, 5))
    for i in range(n):
        kept = np.nonzero(rows[i, :, 5] > 0.5)[0]
        order = kept[np.lexsort((kept, -rows[i, kept, 4]))][:post_n]
        out[i, :len(order), :4] = rows[i, order, :4]
        out[i, :len(order), 4] = 1.0
    return out.reshape(n, -1)


def roi_align(feat, rois, out, scale, sampling):
    """torchvision.ops.roi_align, aligned=False, one feature map [C, H, W] and rois
    [R, 4] in image pixels -> [R, C, out, out].  Bin (ph, pw) averages sampling^2
    bilinear samples at roi_start + (p + (i + 0.5)/sampling) * bin; samples beyond
    [-1, H] x [-1, W] are 0, coordinates below 0 are clamped to 0 and the last row /
    column is replicated (the reference kernel's bilinear_interpolate)."""
    C, H, W = feat.shape
    res = np.zeros((len(rois), C, out, out))
    for r, (x1, y1, x2, y2) in enumerate(rois):
        sw, sh = x1 * scale, y1 * scale
        rw = max(x2 * scale - sw, 1.0)
        rh = max(y2 * scale - sh, 1.0)
        bw, bh = rw / out, rh / out
        for ph in range(out):
            for pw in range(out):
                acc = np.zeros(C)
                for iy in range(sampling):
                    y = sh + ph * bh + (iy + 0.5) * bh / sampling
                    for ix in range(sampling):
                        x = sw + pw * bw + (ix + 0.5) * bw / sampling
                        if y < -1.0 or y > H or x < -1.0 or x > W:
                            continue
                        yy, xx = max(y, 0.0), max(x, 0.0)
                        y0, x0 = int(yy), int(xx)
                        if y0 >= H - 1:
                            y0 = y1_ = H - 1
                            yy = float(y0)
                        else:
                            y1_ = y0 + 1
                        if x0 >= W - 1:
                            x0 = x1_ = W - 1
                            xx = float(x0)
                        else:
                            x1_ = x0 + 1
                        ly, lx = yy - y0, xx - x0
                        hy, hx = 1.0 - ly, 1.0 - lx
                        acc += (hy * hx * feat[:, y0, x0] + hy * lx * feat[:, y0, x1_] +
                                ly * hx * feat[:, y1_, x0] + ly * lx * feat[:, y1_, x1_])
                res[r, :, ph, pw] = acc / (sampling * sampling)
    return res


def roi_levels(rois, k_min, k_max, canonical):
    """MultiScaleRoIAlign's LevelMapper: floor(lvl0 + log2(sqrt(area) / s0) + 1e-6)
    clamped to [k_min, k_max], as an index from k_min (area 0 -> k_min)."""
    s0, lvl0 = canonical
    area = (rois[:, 2] - rois[:, 0]) * (rois[:, 3] - rois[:, 1])
    with np.errstate(divide="ignore"):
        t = np.floor(lvl0 + np.log2(np.sqrt(area) / s0) + 1e-6)
    return (np.clip(t, k_min, k_max) - k_min).astype(np.int64)


def multiscale_roi_align(feats, props, out, sampling, canonical, img_hw):
    """MultiScaleRoIAlign over feature maps finest first (P2..P5): each map's scale
    is 2^round(log2(feature / image)); each proposal is pooled from the map its
    LevelMapper level names.  feats [N, C, H_l, W_l]; props [N, R*5] (rpn_merge).
    Output [N*R, C, out, out] (one row per proposal, frame-major)."""
    n = props.shape[0]
    rois = props.reshape(n, -1, 5)[..., :4]
    R = rois.shape[1]
    scales = [2.0 ** round(math.log2(f.shape[2] / img_hw[0])) for f in feats]
    k_min, k_max = int(round(-math.log2(scales[0]))), int(round(-math.log2(scales[-1])))
    C = feats[0].shape[1]
    res = np.zeros((n * R, C, out, out))
    for i in range(n):
        lv = roi_levels(rois[i], k_min, k_max, canonical)
        for l, f in enumerate(feats):
            idx = np.nonzero(lv == l)[0]
            if len(idx):
                res[i * R + idx] = roi_align(f[i], rois[i, idx], out, scales[l], sampling)
    return res


def box_post(cls, box, props, classes, weights, img_hw):
    """Fast R-CNN box decode (RoIHeads.postprocess_detections up to its score
    threshold): per proposal the class deltas decoded against it (BoxCoder(weights)),
    clipped to the image; class probabilities = softmax of the logits; background
    (class 0) dropped.  cls [N*R, classes], box [N*R, classes*4], props [N, R*5].
    Output [N, R*(classes-1)*6]: rows (x1, y1, x2, y2, score, label) in (proposal,
    class) order; rows of a missing proposal (valid flag 0) score -1."""
    n = props.shape[0]
    p = props.reshape(n, -1, 5)
    R = p.shape[1]
    lg = cls.reshape(n, R, classes)
    e = np.exp(lg - lg.max(axis=-1, keepdims=True))
    prob = e / e.sum(axis=-1, keepdims=True)
    d = box.reshape(n, R, classes, 4)
    b = clip_boxes(box_decode(d, p[:, :, None, :4], weights), img_hw)
    out = np.zeros((n, R, classes - 1, 6))
    out[..., :4] = b[:, :, 1:]
    out[..., 4] = np.where(p[:, :, 4:5] > 0.5, prob[:, :, 1:], -1.0)
    out[..., 5] = np.arange(1, classes)[None, None, :]
    return out.reshape(n, -1)


# ----------------------------------------------------------------------------
# Final detection post-processing: candidates -> top-k -> NMS
# ----------------------------------------------------------------------------

def det_candidates(x, fmt, fields, score_thresh, min_size):
    """Candidate detections (reading R22): x [N, n*fields] rows ->
    [N, n*6] rows (x1, y1, x2, y2, score, label); a dropped row scores -1.
      fmt 0, Fast R-CNN box_post rows (x1, y1, x2, y2, p, label): taken as they are
         (torchvision RoIHeads.postprocess_detections scores every (proposal, class));
      fmt 1, YOLO decode rows (cx, cy, w, h, obj, cls_0 .. cls_{C-1}): box (cx - w/2,
         cy - h/2, cx + w/2, cy + h/2), score obj * max_k cls_k, label the first argmax k
         (one label per box: darknet/ultralytics single-label detection);
      fmt 2, SSD decode rows (x1, y1, x2, y2, best_fg, p_0 .. p_{C-1}): score
         max_{k>=1} p_k, label the first argmax k >= 1 (one label per box).
    A row is kept iff score > score_thresh and both sides >= min_size
    (torchvision: scores > box_score_thresh, then remove_small_boxes)."""
    n = x.shape[0]
    r = x.reshape(n, -1, fields).astype(np.float64)
    out = np.zeros(r.shape[:2] + (6,))
    if fmt == 0:
        out[...] = r[..., :6]
    elif fmt == 1:
        cls = r[..., 5:]
        k = np.argmax(cls, axis=-1)
        out[..., 0] = r[..., 0] - r[..., 2] / 2
        out[..., 1] = r[..., 1] - r[..., 3] / 2
        out[..., 2] = r[..., 0] + r[..., 2] / 2
        out[..., 3] = r[..., 1] + r[..., 3] / 2
        out[..., 4] = r[..., 4] * np.take_along_axis(cls, k[..., None], -1)[..., 0]
        out[..., 5] = k
    else:
        fg = r[..., 6:]
        k = np.argmax(fg, axis=-1)
        out[..., :4] = r[..., :4]
        out[..., 4] = np.take_along_axis(fg, k[..., None], -1)[..., 0]
        out[..., 5] = k + 1
    w = out[..., 2] - out[..., 0]
    h = out[..., 3] - out[..., 1]
    keep = (out[..., 4] > score_thresh) & (w >= min_size) & (h >= min_size)
    out[..., 4] = np.where(keep, out[..., 4], -1.0)
    return out.reshape(n, -1)


def det_nms(top, iou_thresh, max_det):
    """Greedy batched NMS over score-ranked candidates (torchvision batched_nms: boxes
    of different labels never suppress each other).  top: topk_rows output over
    det_candidates rows, [N, K*7] rows (index, x1, y1, x2, y2, score, label) in
    descending score order.  A row is visited unless its index is -1 or its score is
    negative (dropped); it is kept unless an already kept row of the same label
    overlaps it with IoU > iou_thresh (IoU = inter / (area_i + area_j - inter); 0/0
    never suppresses).  Output [N, max_det*6]: the first max_det kept rows in visiting
    order as (x1, y1, x2, y2, score, label); missing rows (0, 0, 0, 0, -1, 0)."""
    n = top.shape[0]
    t = top.reshape(n, -1, 7)
    out = np.zeros((n, max_det, 6))
    out[:, :, 4] = -1.0
    for f in range(n):
        kept = []
        for row in t[f]:
            if row[0] < 0 or row[5] < 0:
                continue
            b = row[1:5]
            sup = False
            for kb in kept:
                if kb[5] != row[6]:
                    continue
                iw = max(0.0, min(b[2], kb[2]) - max(b[0], kb[0]))
                ih = max(0.0, min(b[3], kb[3]) - max(b[1], kb[1]))
                inter = iw * ih
                den = (b[2] - b[0]) * (b[3] - b[1]) + (kb[2] - kb[0]) * (kb[3] - kb[1]) - inter
                with np.errstate(invalid="ignore", divide="ignore"):
                    iou = np.float64(inter) / np.float64(den)
                if iou > iou_thresh:
                    sup = True
                    break
            if not sup:
                kept.append(np.concatenate([b, row[5:7]]))
                if len(kept) == max_det:
                    break
        if kept:
            out[f, :len(kept)] = np.array(kept)
    return out.reshape(n, -1)


def out_shape(layer, in_shapes):
    """(C, H, W) or (F,) of a layer's output given its inputs' shapes (oracle's own)."""
    op = layer["op"]
    s0 = in_shapes[0]
    if op == "conv":
        _, h, w = s0
        return (layer["cout"], conv_out_size(h, layer["k"][0], layer["s"][0], layer["p"][0], layer["d"][0]),
                conv_out_size(w, layer["k"][1], layer["s"][1], layer["p"][1], layer["d"][1]))
    if op in ("bn", "relu", "leaky", "add"):
        return s0
    if op == "maxpool":
        c, h, w = s0
        if layer.get("darknet"):
            return (c, (h - 1) // layer["s"][0] + 1, (w - 1) // layer["s"][1] + 1)
        return (c, pool_out_size(h, layer["k"][0], layer["s"][0], layer["p"][0], layer["d"][0], layer["ceil"]),
                pool_out_size(w, layer["k"][1], layer["s"][1], layer["p"][1], layer["d"][1], layer["ceil"]))
    if op == "gap":
        return (s0[0],) + tuple(layer["out"])
    if op == "concat":
        return (sum(s[0] for s in in_shapes),) + tuple(s0[1:])
    if op == "upsample":
        return (s0[0], s0[1] * layer["scale"], s0[2] * layer["scale"])
    if op == "flatten":
        return (int(math.prod(s0)),)
    if op == "linear":
        return (layer["fout"],)
    if op == "yolo":
        c, h, w = s0
        return (len(layer["anchors"]) * h * w * (5 + layer["classes"]),)
    if op == "topk":
        return (layer["k"] * (layer["fields"] + 1),)
    if op == "l2norm":
        return s0
    if op == "ssd_decode":
        c, h, w = s0
        return (len(layer["wh"]) * h * w * (5 + layer["classes"]),)
    if op == "rpn_level":
        c, h, w = s0
        return (min(layer["pre_n"], c * h * w) * 6,)
    if op == "rpn_merge":
        return (layer["post_n"] * 5,)
    if op == "roi_align":
        return (in_shapes[1][0], layer["out"], layer["out"])     # per proposal
    if op == "box_post":
        return (in_shapes[2][0] // 5 * (layer["classes"] - 1) * 6,)
    if op == "det_cand":
        return (s0[0] // layer["fields"] * 6,)
    if op == "det_nms":
        return (layer["max_det"] * 6,)
    raise ValueError(f"unknown op {op}")
