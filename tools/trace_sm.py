"""Per-CTA timeline of one problem in a GEMEL_TRACE_DIR capture: how a CTA's time
splits between consecutive tiles (developer tool)."""
import json
import sys

import numpy as np

d = json.load(open(sys.argv[1] + "/plan.json"))
li, pi = int(sys.argv[2]), int(sys.argv[3])
L = d["plan"]["launches"][li]
raw = np.fromfile(f"{sys.argv[1]}/launch{li}.bin", dtype=np.uint64).reshape(-1, 16).astype(np.int64)
t0 = raw[:, 0].min()
begin = 0
for i, p in enumerate(L["problems"]):
    n = -(-p["M"] // 128) * -(-p["N"] // p["bn"]) * p.get("ksplit", 1)
    if i == pi:
        break
    begin += n
r = raw[begin:begin + n]
t = (r[:, :8] - t0) / 1e3
cta = r[:, 8]
print(f"problem {pi}: {n} tiles, CTAs used {len(set(cta.tolist()))}")
for c in sorted(set(cta.tolist()))[:3]:
    idx = np.where(cta == c)[0]
    idx = idx[np.argsort(t[idx, 0])]
    print(f"CTA {c}: {len(idx)} tiles")
    for k in idx[:8]:
        print("  grab %.1f ready %.1f lastTMA %.1f land %.1f lastMMA %.1f acc %.1f st %.1f pub %.1f" % tuple(t[k]))
