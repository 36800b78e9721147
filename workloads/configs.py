"""Workload configurations (BASELINE.json ``configs``; compositions from SURVEY.md §8).

A config is a list of queries -- (model name, camera stream id) -- plus the
frame resolution and the per-stream batch B.  One query per stream, as in the
paper's edge workloads where each query runs one DNN on one feed.

  cfg1: Tiny-A + Tiny-B, 2 streams, B=2, 32x32 (configs[0], oracle in seconds)
  cfg2: ResNet-18 + ResNet-34 + ResNet-50, 3 streams, B=8, 224x224 (configs[1];
        the bench workload)
  cfg3: 3x VGG-16 + 3x VGG-19 (alternating streams), B=8, 224x224 (configs[2])
"""
from __future__ import annotations

CONFIGS = {
    1: {"name": "cfg1_tiny", "queries": [("tiny_a", 0), ("tiny_b", 1)], "res": 32, "batch": 2},
    2: {"name": "cfg2_resnet18_34_50", "queries": [("resnet18", 0), ("resnet34", 1), ("resnet50", 2)],
        "res": 224, "batch": 8},
    3: {"name": "cfg3_vgg16x3_vgg19x3",
        "queries": [("vgg16", 0), ("vgg19", 1), ("vgg16", 2), ("vgg19", 3), ("vgg16", 4), ("vgg19", 5)],
        "res": 224, "batch": 8},
}


def weight_key(cfg, query_index):
    """Philox key prefix for a query's weights: (cfg, query)."""
    return (cfg, query_index)
