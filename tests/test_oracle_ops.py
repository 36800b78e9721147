"""Pins for oracle/ops.py: special cases that reduce to library routines
(torch.nn.functional in fp64 on CPU -- a different implementation), closed
forms and brute force.  The GPU path never calls torch compute."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import ops

RTOL = 1e-12


def _t(x):
    return torch.from_numpy(np.ascontiguousarray(x))


def _close(a, b, tol=RTOL):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    err = np.max(np.abs(a - b) / (np.abs(b) + 1e-9)) if a.size else 0.0
    assert err <= tol * 1e3 or np.max(np.abs(a - b)) <= tol * max(1.0, np.max(np.abs(b))), err


CONV_CASES = [
    # n, cin, cout, h, w, k, s, p, d, groups, bias
    (2, 3, 8, 9, 11, (3, 3), (1, 1), (1, 1), (1, 1), 1, True),
    (1, 4, 6, 10, 10, (7, 7), (2, 2), (3, 3), (1, 1), 1, False),
    (2, 8, 4, 7, 7, (1, 1), (2, 2), (0, 0), (1, 1), 1, False),
    (1, 6, 6, 13, 12, (3, 3), (1, 1), (6, 6), (6, 6), 1, True),     # SSD-style dilation 6
    (2, 6, 4, 8, 9, (3, 3), (2, 1), (1, 0), (1, 2), 2, True),       # groups, asymmetric
    (1, 3, 5, 11, 11, (11, 11), (4, 4), (2, 2), (1, 1), 1, True),   # AlexNet stem
]


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv2d_matches_torch(case):
    n, cin, cout, h, w, k, s, p, d, g, bias = case
    rng = np.random.default_rng(0)
    x = rng.standard_normal((n, cin, h, w))
    wt = rng.standard_normal((cout, cin // g) + k)
    b = rng.standard_normal(cout) if bias else None
    y = ops.conv2d(x, wt, b, s, p, d, g)
    ref = F.conv2d(_t(x), _t(wt), None if b is None else _t(b), s, p, d, g).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-10, atol=1e-11)


def test_conv1x1_is_matmul():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((3, 5, 4, 6))
    w = rng.standard_normal((7, 5, 1, 1))
    y = ops.conv2d(x, w, None, (1, 1), (0, 0), (1, 1))
    ref = np.einsum("nchw,oc->nohw", x, w[:, :, 0, 0])
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)


def test_conv_brute_force_tiny():
    """Literal six-fold loop of the definition on a tiny case."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal((1, 2, 5, 4))
    w = rng.standard_normal((3, 2, 3, 2))
    b = rng.standard_normal(3)
    s, p, d = (2, 1), (1, 1), (1, 2)
    y = ops.conv2d(x, w, b, s, p, d)
    ho = (5 + 2 - 1 * 2 - 1) // 2 + 1
    wo = (4 + 2 - 2 * 1 - 1) // 1 + 1
    assert y.shape == (1, 3, ho, wo)
    for co in range(3):
        for i in range(ho):
            for j in range(wo):
                acc = b[co]
                for ci in range(2):
                    for r in range(3):
                        for t in range(2):
                            ih, iw = i * 2 - 1 + r, j - 1 + 2 * t
                            if 0 <= ih < 5 and 0 <= iw < 4:
                                acc += w[co, ci, r, t] * x[0, ci, ih, iw]
                assert abs(y[0, co, i, j] - acc) < 1e-12


@pytest.mark.parametrize("k,s,p,ceil", [((3, 3), (2, 2), (1, 1), False), ((2, 2), (2, 2), (0, 0), False),
                                         ((3, 3), (2, 2), (0, 0), True), ((2, 2), (2, 2), (0, 0), True),
                                         ((3, 3), (1, 1), (1, 1), False)])
@pytest.mark.parametrize("hw", [(7, 7), (8, 9), (75, 75), (13, 13)])
def test_maxpool_matches_torch(k, s, p, ceil, hw):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 3) + hw)
    y = ops.maxpool2d(x, k, s, p, (1, 1), ceil)
    ref = F.max_pool2d(_t(x), k, s, p, 1, ceil_mode=ceil).numpy()
    np.testing.assert_array_equal(y, ref)


def test_darknet_maxpool_is_right_bottom_pad():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((1, 2, 13, 13)) - 0.5
    y = ops.maxpool2d(x, (2, 2), (1, 1), (0, 0), darknet=True)
    ref = F.max_pool2d(F.pad(_t(x), (0, 1, 0, 1), value=-np.inf), 2, 1).numpy()
    assert y.shape == (1, 2, 13, 13)
    np.testing.assert_array_equal(y, ref)


@pytest.mark.parametrize("hw,out", [((7, 7), (1, 1)), ((7, 7), (7, 7)), ((10, 13), (3, 4)), ((1, 1), (7, 7)),
                                    ((13, 13), (6, 6))])
def test_adaptive_avgpool_matches_torch(hw, out):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 3) + hw)
    y = ops.adaptive_avgpool2d(x, out)
    ref = F.adaptive_avg_pool2d(_t(x), out).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-13)


def test_batchnorm_matches_torch():
    rng = np.random.default_rng(6)
    x = rng.standard_normal((2, 5, 3, 4))
    g, b, m = rng.standard_normal(5), rng.standard_normal(5), rng.standard_normal(5)
    v = rng.uniform(0.5, 2, 5)
    y = ops.batchnorm(x, g, b, m, v, 1e-5)
    ref = F.batch_norm(_t(x), _t(m), _t(v), _t(g), _t(b), False, 0.1, 1e-5).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)


def test_linear_relu_leaky_upsample_flatten():
    rng = np.random.default_rng(7)
    x = rng.standard_normal((3, 10))
    w, b = rng.standard_normal((4, 10)), rng.standard_normal(4)
    np.testing.assert_allclose(ops.linear(x, w, b), F.linear(_t(x), _t(w), _t(b)).numpy(), rtol=1e-12)
    np.testing.assert_array_equal(ops.relu(x), F.relu(_t(x)).numpy())
    np.testing.assert_allclose(ops.leaky_relu(x, 0.1), F.leaky_relu(_t(x), 0.1).numpy(), rtol=1e-15)
    y = rng.standard_normal((2, 3, 4, 5))
    np.testing.assert_array_equal(ops.upsample_nearest(y, 2),
                                  F.interpolate(_t(y), scale_factor=2, mode="nearest").numpy())
    np.testing.assert_array_equal(ops.flatten(y), torch.flatten(_t(y), 1).numpy())


def test_preprocess_closed_form():
    f = np.zeros((1, 2, 2, 3), np.uint8)
    f[0, 0, 0] = (0, 0, 0)
    f[0, 0, 1] = (255, 255, 255)
    f[0, 1, 0] = (51, 102, 153)
    x = ops.preprocess(f)
    assert x.shape == (1, 3, 2, 2)
    np.testing.assert_allclose(x[0, :, 0, 0], -ops.IMAGENET_MEAN / ops.IMAGENET_STD, rtol=1e-15)
    np.testing.assert_allclose(x[0, :, 0, 1], (1 - ops.IMAGENET_MEAN) / ops.IMAGENET_STD, rtol=1e-15)
    np.testing.assert_allclose(x[0, 0, 1, 0], (0.2 - 0.485) / 0.229, rtol=1e-14)


def test_out_shapes_match_torch_modules():
    x = torch.zeros(1, 3, 224, 224, dtype=torch.float64)
    assert ops.conv_out_size(224, 7, 2, 3, 1) == F.conv2d(x, torch.zeros(1, 3, 7, 7, dtype=torch.float64),
                                                          stride=2, padding=3).shape[-1]
    assert ops.pool_out_size(75, 3, 2, 0, 1, True) == F.max_pool2d(torch.zeros(1, 1, 75, 75), 3, 2,
                                                                   ceil_mode=True).shape[-1]


def test_topk_rows_brute_force_and_ties():
    """Top-k by one column, ties by lower row index: against a brute-force ranking."""
    rng = np.random.default_rng(5)
    fields, n, k = 6, 50, 7
    x = rng.integers(0, 5, size=(3, n * fields)).astype(np.float64)   # many exact ties
    y = ops.topk_rows(x, k, fields, 2).reshape(3, k, fields + 1)
    for i in range(3):
        rows = x[i].reshape(n, fields)
        ranked = sorted(range(n), key=lambda r: (-rows[r, 2], r))[:k]
        assert [int(v) for v in y[i, :, 0]] == ranked
        np.testing.assert_array_equal(y[i, :, 1:], rows[ranked])
    short = ops.topk_rows(x[:, :3 * fields], 5, fields, 2).reshape(3, 5, fields + 1)
    assert (short[:, 3:, 0] == -1).all() and (short[:, 3:, 1:] == 0).all()
