"""Pins of the oracle's final detection post-processing (DESIGN.md
reading R22): oracle.ops.det_candidates -> topk_rows -> det_nms against torchvision
(batched_nms; RoIHeads.postprocess_detections end to end) and hand-worked cases."""
import numpy as np
import pytest
import torch

from oracle import ops

tv = pytest.importorskip("torchvision")


def _pipeline(rows6, thresh, min_size, iou, max_det, k=None):
    """Fast R-CNN-format rows [N, n*6] -> final detections [N, max_det, 6]."""
    n = rows6.shape[1] // 6
    cand = ops.det_candidates(rows6, 0, 6, thresh, min_size)
    top = ops.topk_rows(cand, k or n, 6, 4)
    return ops.det_nms(top, iou, max_det).reshape(rows6.shape[0], max_det, 6)


def _random_boxes(rng, n, size=100.0):
    xy = rng.uniform(0, size, (n, 2))
    wh = rng.uniform(1, size / 3, (n, 2))
    return np.concatenate([xy, xy + wh], axis=1)


@pytest.mark.parametrize("seed", range(6))
def test_det_nms_equals_torchvision_batched_nms(seed):
    rng = np.random.default_rng(seed)
    n = 300
    boxes = _random_boxes(rng, n)
    scores = rng.permutation(n).astype(np.float64) / n + 0.5     # distinct, positive
    labels = rng.integers(0, 4, n).astype(np.float64)
    rows = np.concatenate([boxes, scores[:, None], labels[:, None]], axis=1).reshape(1, -1)
    got = _pipeline(rows, 0.0, 0.0, 0.5, n)[0]
    keep = tv.ops.batched_nms(torch.from_numpy(boxes), torch.from_numpy(scores), torch.from_numpy(labels).long(),
                              0.5).numpy()
    n_kept = int((got[:, 4] >= 0).sum())
    assert n_kept == len(keep)
    np.testing.assert_array_equal(got[:n_kept, :4], boxes[keep])
    np.testing.assert_array_equal(got[:n_kept, 4], scores[keep])
    np.testing.assert_array_equal(got[:n_kept, 5], labels[keep])
    assert np.all(got[n_kept:, 4] == -1.0)


@pytest.mark.parametrize("seed", range(3))
def test_fast_rcnn_postprocess_equals_torchvision_roi_heads(seed):
    """box_post -> det_candidates(fmt 0) -> topk (all rows) -> det_nms reproduces torchvision
    RoIHeads.postprocess_detections (score > 0.05, min size 1e-2, batched NMS 0.5, 100)."""
    from torchvision.models.detection.roi_heads import RoIHeads
    rng = np.random.default_rng(100 + seed)
    R, C, H, W = 200, 11, 300, 400
    props = _random_boxes(rng, R, 250.0)
    logits = rng.normal(0, 3, (R, C))
    deltas = rng.normal(0, 0.3, (R, C * 4))
    heads = RoIHeads(None, None, None, 0.5, 0.5, 512, 0.25, None, 0.05, 0.5, 100)
    tb, ts, tl = heads.postprocess_detections(torch.from_numpy(logits), torch.from_numpy(deltas),
                                              [torch.from_numpy(props)], [(H, W)])
    tb, ts, tl = tb[0].numpy(), ts[0].numpy(), tl[0].numpy()
    p5 = np.concatenate([props, np.ones((R, 1))], axis=1).reshape(1, -1)
    rows = ops.box_post(logits, deltas, p5, C, (10.0, 10.0, 5.0, 5.0), (H, W))
    got = _pipeline(rows, 0.05, 1e-2, 0.5, 100)[0]
    n_kept = int((got[:, 4] >= 0).sum())
    assert n_kept == len(ts) > 0
    np.testing.assert_allclose(got[:n_kept, :4], tb, rtol=0, atol=1e-9)
    np.testing.assert_allclose(got[:n_kept, 4], ts, rtol=1e-12, atol=0)
    np.testing.assert_array_equal(got[:n_kept, 5], tl)


def test_yolo_candidates_closed_form():
    """YOLO rows (cx, cy, w, h, obj, cls...): corners, obj * best class, first argmax."""
    rows = np.array([[10, 20, 4, 6, 0.5, 0.2, 0.9, 0.9],      # classes tie at 1 and 2 -> label 1
                     [50, 50, 10, 10, 0.1, 0.5, 0.4, 0.3],   # 0.05 <= thresh 0.1 -> dropped
                     [30, 40, 2, 2, 1.0, 0.0, 0.0, 0.25]], np.float64).reshape(1, -1)
    c = ops.det_candidates(rows, 1, 8, 0.1, 0.0).reshape(3, 6)
    np.testing.assert_allclose(c[0], [8, 17, 12, 23, 0.45, 1])
    assert c[1, 4] == -1.0 and c[1, 5] == 0
    np.testing.assert_allclose(c[2], [29, 39, 31, 41, 0.25, 2])


def test_ssd_candidates_closed_form():
    """SSD rows (x1, y1, x2, y2, best, p_0 .. p_{C-1}): best class >= 1, its first argmax."""
    rows = np.array([[0, 0, 5, 5, 0.6, 0.1, 0.6, 0.3],
                     [1, 1, 1.005, 3, 0.5, 0.0, 0.5, 0.5]], np.float64).reshape(1, -1)
    c = ops.det_candidates(rows, 2, 8, 0.01, 1e-2).reshape(2, 6)
    np.testing.assert_allclose(c[0], [0, 0, 5, 5, 0.6, 1])
    assert c[1, 4] == -1.0 and c[1, 5] == 1        # width 0.005 < min size: dropped, label still first argmax


def test_det_nms_edge_cases():
    # identical boxes of one label: only the best survives; another label is untouched;
    # IoU exactly at the threshold does not suppress; zero-area boxes never suppress (0/0)
    b = [[0, 0, 10, 10, 0.9, 1], [0, 0, 10, 10, 0.8, 1], [0, 0, 10, 10, 0.7, 2],
         [0, 0, 10, 5, 0.6, 1],                      # IoU with the first = 50/100 = 0.5 -> kept at 0.5
         [3, 3, 3, 3, 0.5, 3], [3, 3, 3, 3, 0.4, 3]]
    rows = np.array(b, np.float64).reshape(1, -1)
    got = _pipeline(rows, 0.0, 0.0, 0.5, 10)[0]
    np.testing.assert_array_equal(got[:5, 4], [0.9, 0.7, 0.6, 0.5, 0.4])
    assert np.all(got[5:, 4] == -1.0) and np.all(got[5:, :4] == 0)
    # max_det truncates in visiting order
    got2 = _pipeline(rows, 0.0, 0.0, 0.5, 2)[0]
    np.testing.assert_array_equal(got2[:, 4], [0.9, 0.7])
    # every candidate dropped by the threshold: all rows padding
    got3 = _pipeline(rows, 0.95, 0.0, 0.5, 4)[0]
    assert np.all(got3[:, 4] == -1.0)
    # a pre-NMS cap (topk k) keeps only the k best candidates: 0.9 and 0.8, and 0.8 is
    # suppressed by 0.9 (same box, same label)
    got4 = _pipeline(rows, 0.0, 0.0, 0.5, 10, k=2)[0]
    assert got4[0, 4] == 0.9 and np.all(got4[1:, 4] == -1.0)
