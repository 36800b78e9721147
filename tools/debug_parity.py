"""Developer tool: teacher-forced per-value errors of one small config, with bad-element locations."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import merge as om  # noqa: E402
from paper_2201_07705_b200.engine import MergedWorkload  # noqa: E402
from tests.gpu_util import like, oracle_layer, rel_err, to_nchw  # noqa: E402
from oracle import model as omodel, ops  # noqa: E402
from workloads import synth, zoo  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["resnet18", "resnet34", "resnet50"]
res = int(sys.argv[2]) if len(sys.argv) > 2 else 64
B = int(sys.argv[3]) if len(sys.argv) > 3 else 2
models = [zoo.build(n) for n in names]
params = [synth.params(m, 2, q) for q, m in enumerate(models)]
wl = MergedWorkload([(m, p, i) for i, (m, p) in enumerate(zip(models, params))], (res, res), B)
fr = {i: synth.frames(2, i, B, res, res) for i in range(len(models))}
outs = wl.alloc_outputs()
wl.infer({i: torch.from_numpy(f).cuda() for i, f in fr.items()}, outs)
torch.cuda.synchronize()
mp = om.merged_params(models, params, wl.merge_config)
for mid, layers in enumerate(models):
    stored = omodel.storage_points(layers)
    x = ops.preprocess(fr[mid])
    vals = {-1: omodel.round_bf16(x)}
    for i, l in enumerate(layers):
        y = oracle_layer(l, mp[mid][i], [vals[j] for j in l["in"]])
        if stored[i] or i == len(layers) - 1:
            g = like(to_nchw(wl.read_value(mid, i)), y)
            e = rel_err(g, y)
            if e > 0.02:
                bad = np.argwhere(np.abs(g - y) / (np.abs(y) + 1e-3) > 0.02)
                print(f"{names[mid]} pos {i} {l['op']} shape {y.shape} err {e:.3g} nbad {len(bad)} first {bad[:6].tolist()}"
                      f" rows(n) {sorted(set(bad[:, 0].tolist()))[:8]} chans {sorted(set(bad[:, 1].tolist()))[:12]}")
            vals[i] = g
        else:
            vals[i] = y
print("plan", wl.plan)
