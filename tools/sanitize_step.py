"""Developer check (run under compute-sanitizer): one merged step of a small workload
through the C ABI, launches issued directly (profiling mode, no graph).

    compute-sanitizer --tool memcheck python tools/sanitize_step.py cfg1|cfg2b1|frcnn64
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import merge as om  # noqa: E402  (merge configuration only)
from paper_2201_07705_b200.engine import MergedWorkload  # noqa: E402
from workloads import synth, zoo  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
names, res, batch = {"cfg1": (["tiny_a", "tiny_b"], 32, 2),
                     "cfg2b1": (["resnet18", "resnet34", "resnet50"], 224, 1),
                     "frcnn64": (["frcnn_r50_fpn", "frcnn_r50_fpn"], 64, 2),
                     "yolo256": (["yolov3", "yolov3"], 256, 1)}[case]
models = [zoo.build(n) for n in names]
params = [synth.params(m, 9, q) for q, m in enumerate(models)]
merge = om.cross_model_groups(om.find_shareable(models))
wl = MergedWorkload([(m, p, q) for q, (m, p) in enumerate(zip(models, params))], (res, res), batch, merge=merge)
frames = {q: torch.from_numpy(synth.frames(9, q, batch, res, res)).cuda() for q in range(len(models))}
outs = wl.alloc_outputs()
wl.set_profiling(True)
wl.infer(frames, outs)
torch.cuda.synchronize()
wl.set_profiling(False)
wl.infer(frames, outs)       # the captured graph too
torch.cuda.synchronize()
print("ok", case, wl.plan["n_launches"])
