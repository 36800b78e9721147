"""Developer tool: per-launch device time of one profiled step (CUDA events per
launch, no graph) for a config, summed per kernel kind.
    CFG=4 python tools/launch_breakdown.py"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2201_07705_b200.engine import MergedWorkload  # noqa: E402
from workloads import configs, synth, zoo  # noqa: E402

cfg_id = int(os.environ.get("CFG", "4"))
cfg = configs.CONFIGS[cfg_id]
qs = []
for q, (name, sid) in enumerate(cfg["queries"]):
    l = zoo.build(name)
    qs.append((l, synth.params(l, cfg_id, q), sid))
wl = MergedWorkload(qs, {s: (configs.stream_res(cfg, s),) * 2 for _, s in cfg["queries"]}, cfg["batch"],
                    merge=os.environ.get("MERGE", "cross"))
frames = {s: torch.from_numpy(synth.frames(cfg_id, s, cfg["batch"], configs.stream_res(cfg, s),
                                           configs.stream_res(cfg, s))).cuda()
          for _, s in cfg["queries"]}
outs = wl.alloc_outputs()
wl.set_profiling(True)
for _ in range(3):
    wl.infer(frames, outs)
torch.cuda.synchronize()
ll = wl.launch_list()
agg = defaultdict(lambda: [0, 0.0])
for i, L in enumerate(ll):
    agg[L["kind"]][0] += 1
    agg[L["kind"]][1] += L["ms"]
    print(f"{i:3d} {L['kind']:12s} lvl {L['level']:3d} {L['ms']*1e3:9.1f} us  GFLOP {L['flops']/1e9:8.1f}  MB {L['bytes']/1e6:8.1f}")
tot = sum(v[1] for v in agg.values())
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:12s} {n:4d} launches {ms*1e3:9.1f} us  {ms/tot:6.1%}")
