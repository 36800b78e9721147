"""Summarise a GEMEL_TRACE_DIR capture: per-problem timings of a GEMM launch.

Per tile (ns, globaltimer): 0 grab, 1 deps ready, 2 last TMA issued, 3 first
stage landed (MMA), 4 last MMA issued, 5 accumulator ready (epilogue),
6 stores complete, 7 published.
"""
import json
import sys

import numpy as np

d = json.load(open(sys.argv[1] + "/plan.json"))
li = int(sys.argv[2]) if len(sys.argv) > 2 else 3
nshow = int(sys.argv[3]) if len(sys.argv) > 3 else 100
L = d["plan"]["launches"][li]
raw = np.fromfile(f"{sys.argv[1]}/launch{li}.bin", dtype=np.uint64).reshape(-1, 16).astype(np.int64)
t = raw[:, :8] - raw[:, 0].min()
span = t[:, 7].max() / 1e3
print(f"launch {li}: span {span:.1f} us, tiles {len(t)}")
print("  i mem     M    N     K  bn ks tiles | ready0  done  | deps  issue  1st-land  mma->acc  epi  store->pub (us, mean)")
begin = 0
for i, p in enumerate(L["problems"]):
    mt = -(-p["M"] // 128); nt = -(-p["N"] // p["bn"]); ks = p.get("ksplit", 1); n = mt * nt * ks
    s = t[begin:begin + n] / 1e3
    begin += n
    if i < nshow:
        print("%3d %d %6d %4d %5d %3d %2d %4d | %6.1f %6.1f | %5.1f %5.1f %6.1f %6.1f %6.1f %6.1f" % (
            i, len(p["members"]), p["M"], p["N"], p["K"], p["bn"], ks, n, s[:, 1].min(), s[:, 7].max(),
            (s[:, 1] - s[:, 0]).mean(), (s[:, 2] - s[:, 1]).mean(), (s[:, 3] - s[:, 1]).mean(),
            (s[:, 5] - s[:, 4]).mean(), (s[:, 6] - s[:, 5]).mean(), (s[:, 7] - s[:, 6]).mean()))
busy = (t[:, 7] - t[:, 1]).sum() / 1e3
print("sum(tile ready->published) / (148*span) = %.2f" % (busy / (148 * span)))
