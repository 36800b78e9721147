"""Developer tool: per-tile timestamps of one cfg step (GEMEL_TRACE_DIR) + plan dump."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace"
os.makedirs(out, exist_ok=True)
os.environ["GEMEL_TRACE_DIR"] = out
import torch  # noqa: E402

from paper_2201_07705_b200 import gemel as G  # noqa: E402
from paper_2201_07705_b200.engine import MergedWorkload  # noqa: E402
from workloads import configs, synth, zoo  # noqa: E402

cfg_id = int(os.environ.get("CFG", "2"))
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
json.dump({"plan": G.gemel_plan_dump(wl.ctx), "launches": wl.launch_list()}, open(os.path.join(out, "plan.json"), "w"))
print(json.dumps(wl.launch_list()))
