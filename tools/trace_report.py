"""Summarise a GEMEL_TRACE_DIR capture: per-problem timings of the megakernel launch."""
import json
import sys

import numpy as np

d = json.load(open(sys.argv[1] + "/plan.json"))
li = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L = d["plan"]["launches"][li]
t = np.fromfile(f"{sys.argv[1]}/launch{li}.bin", dtype=np.uint64).reshape(-1, 4).astype(np.int64)
t = t - t[:, 0].min()
span = t[:, 3].max() / 1e3
print(f"launch {li}: span {span:.1f} us, tiles {len(t)}")
begin = 0
tot_epi = tot_load = 0
for i, p in enumerate(L["problems"]):
    mt = -(-p["M"] // 128); nt = -(-p["N"] // p["bn"]); n = mt * nt
    s = t[begin:begin + n]; begin += n
    tot_epi += (s[:, 3] - s[:, 2]).sum(); tot_load += (s[:, 2] - s[:, 1]).sum()
    if i < int(sys.argv[3]) if len(sys.argv) > 3 else 100:
        print("%2d %d M%6d N%4d K%5d bn%3d t%4d | grab %7.1f ready %7.1f done %7.1f | wait %5.1f load+mma %5.1f epi %5.1f" % (
            i, len(p["members"]), p["M"], p["N"], p["K"], p["bn"], n, s[:, 0].min() / 1e3, s[:, 1].min() / 1e3,
            s[:, 3].max() / 1e3, (s[:, 1] - s[:, 0]).mean() / 1e3, (s[:, 2] - s[:, 1]).mean() / 1e3,
            (s[:, 3] - s[:, 2]).mean() / 1e3))
print("sum epi / (148*span) = %.2f ; sum deps->acc / (148*span) = %.2f" % (tot_epi / 1e3 / (148 * span), tot_load / 1e3 / (148 * span)))
