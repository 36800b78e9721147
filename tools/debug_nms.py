"""Developer check: device det_nms vs the oracle on cfg4's YOLOv3 query 3 (first mismatch)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import merge as om  # noqa: E402
from oracle import ops  # noqa: E402
from paper_2201_07705_b200.engine import MergedWorkload  # noqa: E402
from workloads import configs, synth, zoo  # noqa: E402

cfg = configs.CONFIGS[4]
names = [n for n, _ in cfg["queries"]]
sids = [s for _, s in cfg["queries"]]
models = [zoo.build(n) for n in names]
params = [synth.params(m, 4, q) for q, m in enumerate(models)]
merge = om.cross_model_groups(om.find_shareable(models))
wl = MergedWorkload([(m, p, s) for m, p, s in zip(models, params, sids)], {s: (608, 608) for s in sids}, 4,
                    merge=merge)
fr = {s: torch.from_numpy(synth.frames(4, s, 4, 608, 608)).cuda() for s in sids}
outs = wl.alloc_outputs()
wl.infer(fr, outs)
torch.cuda.synchronize()
q = int(sys.argv[1]) if len(sys.argv) > 1 else 3
L = models[q]
n = len(L)
top = wl.read_value(q, n - 2).reshape(4, -1).astype(np.float64)
fin = wl.read_value(q, n - 1).reshape(4, -1, 6).astype(np.float64)
ref = ops.det_nms(top, L[-1]["iou"], L[-1]["max_det"]).reshape(4, -1, 6)
for f in range(4):
    d = np.where(np.any(fin[f] != ref[f], axis=1))[0]
    print("frame", f, "kept dev", int((fin[f, :, 4] >= 0).sum()), "ref", int((ref[f, :, 4] >= 0).sum()),
          "first diff row", d[:5])
    if len(d):
        i = d[0]
        print(" dev", fin[f, i], "\n ref", ref[f, i])
        t = top[f].reshape(-1, 7)
        print(" nonfinite in candidates:", int((~np.isfinite(t)).sum()))
        for k in range(max(0, i - 2), i + 1):
            print("  kept", k, fin[f, k], ref[f, k])
