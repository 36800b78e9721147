"""Summarise an ncu CSV (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) of the memory-bound kernels of one step into achieved DRAM
GB/s per kernel against the measured HBM peak (MEASURED_PEAKS.json).
    python tools/summarize_membound.py gpurun_out/mb/cfg4.csv [...] > profiles/r1_membound.json"""
import csv
import io
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
out = {"peak_hbm_gbs": peak, "note": "ncu --clock-control none, one step, cold per-kernel replay", "configs": {}}
for path in sys.argv[1:]:
    text = open(path).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    per = defaultdict(lambda: defaultdict(float))
    for r in rows:
        per[r["ID"]]["name"] = r["Kernel Name"].split("(")[0].split("::")[-1]
        v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1)
        per[r["ID"]][r["Metric Name"]] = v
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        a = agg[d["name"]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    cfg = os.path.splitext(os.path.basename(path))[0]
    out["configs"][cfg] = {k: {"launches": n, "us": round(t * 1e6, 1), "dram_MB": round(b / 1e6, 1),
                               "achieved_gbs": round(b / t / 1e9, 1) if t else None,
                               "frac_of_hbm_peak": round(b / t / 1e9 / peak, 3) if t else None}
                           for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])}
print(json.dumps(out, indent=1))
