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
    raise ValueError(f"unknown op {op}")
