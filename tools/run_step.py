"""Developer tool: run K graph-replayed steps of a config (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2201_07705_b200.engine import MergedWorkload  # noqa: E402
from workloads import configs, synth, zoo  # noqa: E402

cfg_id = int(os.environ.get("CFG", "2"))
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
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
for _ in range(steps):
    wl.infer(frames, outs)
torch.cuda.synchronize()
print("ok", wl.plan["n_launches"])
