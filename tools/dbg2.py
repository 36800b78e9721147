import sys; sys.path.insert(0,'.')
import numpy as np, torch
from oracle import merge as om, model as omodel
from tests.gpu_util import make_queries, like, to_nchw
from workloads import synth
from paper_2201_07705_b200.engine import MergedWorkload
res = int(sys.argv[1]) if len(sys.argv) > 1 else 256
models, params = make_queries(4, ["yolov3","yolov3"])
wl = MergedWorkload([(m,p,s) for m,p,s in zip(models,params,[0,1])], (res,res), 2, merge=sys.argv[2] if len(sys.argv) > 2 else "full")
fr = {s: synth.frames(4, s, 2, res, res) for s in (0,1)}
outs = wl.alloc_outputs(); wl.infer({s: torch.from_numpy(f).cuda() for s,f in fr.items()}, outs); torch.cuda.synchronize()
mp = om.merged_params(models, params, wl.merge_config)
ref = omodel.run(models[0], mp[0], fr[0][:1], emulate_bf16=True)
st = omodel.storage_points(models[0])
for i, l in enumerate(models[0]):
    if not st[i]: continue
    try: g = wl.read_value(0, i)
    except Exception: continue
    gm, rm = np.abs(g[:1]).max(), np.abs(ref[i]).max()
    if i < 20 or gm > 3 * rm or i % 10 == 0: print(i, l["op"], "gpu max %.3g  oracle max %.3g" % (gm, rm))
