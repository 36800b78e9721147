"""Workload configurations (BASELINE.json ``configs``; compositions from SURVEY.md §8).

A config is a list of queries -- (model name, camera stream id) -- plus the
frame resolution and the per-stream batch B.  One query per stream, as in the
paper's edge workloads where each query runs one DNN on one feed.

  cfg1: Tiny-A + Tiny-B, 2 streams, B=2, 32x32 (configs[0], oracle in seconds)
  cfg2: ResNet-18 + ResNet-34 + ResNet-50, 3 streams, B=8, 224x224 (configs[1])
  cfg3: 3x VGG-16 + 3x VGG-19 (alternating streams), B=8, 224x224 (configs[2])
  cfg4: 4x YOLOv3 + 4x Faster R-CNN R50-FPN at 608x608, B=4 (configs[3]; 8 streams;
        the bench workload: the largest single-GPU config)
  cfg5: SURVEY.md §8's 32-stream mix, B=4: R18x3, R34x2, R50x4, R101x2, R152x3, VGG11,
        VGG13, VGG16x4, VGG19x2 at 224x224; YOLOv3x4 and Tiny-YOLOv3x3 at 416x416;
        SSD300x3 at 300x300 (12 distinct architectures; one query per stream)

Merge configurations ("full" = every group in full, "cross" = cross-model groups,
SURVEY.md §8(c-ii)) are built by the library side (engine.cross_model_merge_config)
and, independently, by the oracle (oracle.merge.cross_model_groups); this module
holds no method arithmetic.
"""
from __future__ import annotations

CONFIGS = {
    1: {"name": "cfg1_tiny", "queries": [("tiny_a", 0), ("tiny_b", 1)], "res": 32, "batch": 2},
    2: {"name": "cfg2_resnet18_34_50", "queries": [("resnet18", 0), ("resnet34", 1), ("resnet50", 2)],
        "res": 224, "batch": 8},
    3: {"name": "cfg3_vgg16x3_vgg19x3",
        "queries": [("vgg16", 0), ("vgg19", 1), ("vgg16", 2), ("vgg19", 3), ("vgg16", 4), ("vgg19", 5)],
        "res": 224, "batch": 8},
    4: {"name": "cfg4_yolov3x4_frcnnx4_608",
        "queries": [("yolov3", 0), ("yolov3", 1), ("yolov3", 2), ("yolov3", 3),
                    ("frcnn_r50_fpn", 4), ("frcnn_r50_fpn", 5), ("frcnn_r50_fpn", 6), ("frcnn_r50_fpn", 7)],
        "res": 608, "batch": 4},
    5: {"name": "cfg5_32_streams_mixed",
        "queries": [(n, i) for i, n in enumerate(
            ["resnet18"] * 3 + ["resnet34"] * 2 + ["resnet50"] * 4 + ["resnet101"] * 2 + ["resnet152"] * 3 +
            ["vgg11", "vgg13"] + ["vgg16"] * 4 + ["vgg19"] * 2 + ["yolov3"] * 4 + ["tiny_yolov3"] * 3 +
            ["ssd300"] * 3)],
        "res": 224, "res_of": {"yolov3": 416, "tiny_yolov3": 416, "ssd300": 300}, "batch": 4},
}


def stream_res(cfg, stream):
    """Frame resolution of a stream (its query's model decides)."""
    name = next(n for n, s in cfg["queries"] if s == stream)
    return cfg.get("res_of", {}).get(name, cfg["res"])


def weight_key(cfg, query_index):
    """Philox key prefix for a query's weights: (cfg, query)."""
    return (cfg, query_index)
