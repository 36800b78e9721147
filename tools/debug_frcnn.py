"""Developer probe: a Faster R-CNN pair at a small resolution through the C ABI,
every stored value teacher-forced against the oracle; prints the layers above the
gate and the error pattern of the worst one.
    python tools/debug_frcnn.py 64 [cross|none]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import merge as om
from paper_2201_07705_b200.engine import MergedWorkload
from tests.gpu_util import TOL, make_queries, teacher_forced, to_nchw, oracle_layer, like, rel_err
from workloads import synth

res = int(sys.argv[1]) if len(sys.argv) > 1 else 64
merge = sys.argv[2] if len(sys.argv) > 2 else "cross"
models, params = make_queries(4, ["frcnn_r50_fpn", "frcnn_r50_fpn"])
wl = MergedWorkload([(models[0], params[0], 0), (models[1], params[1], 1)], (res, res), 2, merge=merge)
fr = {s: synth.frames(4, s, 2, res, res) for s in (0, 1)}
outs = wl.alloc_outputs()
wl.infer({s: torch.from_numpy(f).cuda() for s, f in fr.items()}, outs)
torch.cuda.synchronize()
mp = om.merged_params(models, params, wl.merge_config) if merge != "none" else params
L = models[0]
for mid in range(1):
    errs = teacher_forced(wl.read_value, mid, models[mid], mp[mid], fr[mid])
    bad = {i: e for i, e in errs.items() if e > TOL}
    print("model", mid, "compared", len(errs), "above gate:", {i: (L[i]["op"] if i >= 0 else "in", round(e, 4)) for i, e in bad.items()})
    for i in sorted(bad)[:2]:
        l = L[i]
        ins = [to_nchw(wl.read_value(mid, j)) if j >= 0 else None for j in l["in"]]
        ins = [x.reshape(x.shape[0], -1) if x is not None and x.shape[2:] == (1, 1) else x for x in ins]
        p = mp[mid][l.get("tie", i)]
        y = oracle_layer(l, p, ins, (res, res))
        g = like(to_nchw(wl.read_value(mid, i)), y)
        d = np.abs(g - y) > TOL * (np.abs(y) + 1e-3)
        idx = np.argwhere(d)
        print(" layer", i, l["op"], "shape", y.shape, "bad", d.sum(), "of", d.size, "rows", np.unique(idx[:, 0])[:20],
              "cols", np.unique(idx[:, 1])[:40])
        r0 = idx[0][0]
        np.set_printoptions(precision=4, linewidth=200)
        print(" gpu  ", g.reshape(g.shape[0], -1)[r0, 32:72])
        print(" ref  ", y.reshape(y.shape[0], -1)[r0, 32:72])
