"""Developer tool: per-op teacher-forced errors and end-to-end error breakdown for a YOLO pair."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import merge as om  # noqa: E402
from tests.gpu_util import make_queries, normwise_err, oracle_outputs, rel_err, teacher_forced  # noqa: E402
from workloads import synth  # noqa: E402
from paper_2201_07705_b200.engine import MergedWorkload  # noqa: E402

name, res = sys.argv[1], int(sys.argv[2])
models, params = make_queries(4, [name, name])
wl = MergedWorkload([(m, p, s) for m, p, s in zip(models, params, [0, 1])], (res, res), 2, merge="full")
fr = {s: synth.frames(4, s, 2, res, res) for s in (0, 1)}
outs = wl.alloc_outputs()
wl.infer({s: torch.from_numpy(f).cuda() for s, f in fr.items()}, outs)
torch.cuda.synchronize()
outs = {m: o.cpu().numpy().astype(np.float64) for m, o in outs.items()}
mp = om.merged_params(models, params, wl.merge_config)
errs = teacher_forced(wl.read_value, 0, models[0], mp[0], fr[0])
print("teacher-forced:", {k: round(v, 5) for k, v in errs.items()})
ref = oracle_outputs(models, params, wl.merge_config, [fr[0], fr[1]], emulate_bf16=True)
for mid in range(2):
    g, r = outs[mid].reshape(2, -1, 85), ref[mid].reshape(2, -1, 85)
    for f, nm in ((0, "x"), (1, "y"), (2, "w"), (3, "h"), (4, "obj"), (5, "cls")):
        d = np.abs(g[..., f] - r[..., f]) / (np.abs(r[..., f]) + 1e-3)
        print(mid, nm, "max rel %.4f  median %.2e  max|ref| %.3g" % (d.max(), np.median(d), np.abs(r[..., f]).max()))
    print(mid, "normwise", normwise_err(outs[mid], ref[mid]))
from oracle import model as omodel  # noqa: E402
from tests.gpu_util import like, to_nchw  # noqa: E402
ref_all = omodel.run(models[0], mp[0], fr[0], emulate_bf16=True)
st = omodel.storage_points(models[0])
for i, l in enumerate(models[0]):
    if st[i] or l["op"] == "conv":
        try:
            g = like(to_nchw(wl.read_value(0, i)), ref_all[i])
        except Exception:
            continue
        d = np.abs(g - ref_all[i])
        print(i, l["op"], "free-running normwise %.2e  frac elems differing %.4f  max|ref| %.3g" % (
            d.max() / np.abs(ref_all[i]).max(), float((d > 0).mean()), np.abs(ref_all[i]).max()))
