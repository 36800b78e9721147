"""Sum the DRAM traffic of the grouped-GEMM launches of one step from an ncu CSV
(`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
-k regex:gemel_gemm --csv`) and record it in profiles/ncu_traffic.json under
"<workload>:<merge>" (bench.py's roofline.traffic).

    python tools/ncu_traffic.py <csv> <workload> <merge> [json]
"""
import csv
import json
import os
import sys

path, workload, merge = sys.argv[1:4]
out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                         "profiles", "ncu_traffic.json")
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3,
         "nsecond": 1e-9, "ms": 1e-3}
tot = {"dram__bytes_read.sum": 0.0, "dram__bytes_write.sum": 0.0, "gpu__time_duration.sum": 0.0}
launches = 0
for r in rows[1:]:
    if "gemel_gemm" not in r[ki] or r[mi] not in tot:
        continue
    tot[r[mi]] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    launches += r[mi] == "gpu__time_duration.sum"
d = json.load(open(out)) if os.path.exists(out) else {}
d[f"{workload}:{merge}"] = {"gemm_dram_bytes_per_step": tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"],
                            "dram_read_bytes": tot["dram__bytes_read.sum"],
                            "dram_write_bytes": tot["dram__bytes_write.sum"],
                            "gemm_launches": launches, "ncu_gemm_seconds": tot["gpu__time_duration.sum"],
                            "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                                   "--clock-control none -k regex:gemel_gemm, one graph-replayed step "
                                   "(tools/run_step.py 1); cold-cache serialised launches"}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d[f"{workload}:{merge}"]))
