"""Measured pinned host -> device copy bandwidth (the weight-swap roofline's PCIe term):
best of 10 copies of 1 GiB from pinned host memory, CUDA events."""
import json
import sys

import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
best = 0.0
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    d.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    best = max(best, n / (a.elapsed_time(b) * 1e-3) / 1e9)
json.dump({"h2d_pinned_gbs": best, "bytes": n, "how": "best of 10 x 1 GiB pinned->device copies, CUDA events",
           "gpu": torch.cuda.get_device_name()}, sys.stdout)
