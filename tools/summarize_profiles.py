"""Summarise ncu outputs into profiles/<round>_*.{json,txt} (committed evidence).

    python tools/summarize_profiles.py gpurun_out/r1 r1
reads   <dir>/launches*.csv  (ncu --metrics gpu__time_duration.sum --csv; the first match)
        <dir>/prof_*.ncu-rep (ncu --set full captures) and/or
        <dir>/*_raw.csv      (`ncu -i <rep> --page raw --csv` exported on the GPU box)
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

src, tag = sys.argv[1], sys.argv[2]
out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
os.makedirs(out_dir, exist_ok=True)
summary = {"round": tag}

# ---- launch list: per-kernel share of device time
lps = sorted(glob.glob(os.path.join(src, "launches*.csv")))
lp = lps[0] if lps else ""
if lp:
    summary["launch_list"] = os.path.basename(lp)
    rows = list(csv.reader(open(lp)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    seq = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
              "second": 1e6, "s": 1e6}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "").strip()
        agg[name][0] += 1
        agg[name][1] += v
        seq.append((name, v))
    tot = sum(t for _, t in agg.values())
    summary["launches"] = {k: {"count": n, "total_us": round(t, 1), "share": round(t / tot, 4)}
                           for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])}
    with open(os.path.join(out_dir, f"{tag}_launches.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        f.write("# kernel, launches, total_us, share\n")
        for k, d in summary["launches"].items():
            f.write(f"{k}, {d['count']}, {d['total_us']}, {d['share']}\n")
        f.write("\n# launch sequence (us)\n")
        for name, v in seq:
            f.write(f"{name}, {v:.2f}\n")

# ---- full captures
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
caps = []
for rep in sorted(glob.glob(os.path.join(src, "prof_*.ncu-rep")) + glob.glob(os.path.join(src, "*_raw.csv"))):
    if rep.endswith(".csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"report": os.path.basename(rep), "kernel": r[h.index("Kernel Name")] if "Kernel Name" in h else ""}
        for w in WANT:
            for i, x in enumerate(h):
                if x.endswith(w) or x == w:
                    d[w] = f"{r[i]} {units[i]}".strip()
                    break
        caps.append(d)
summary["ncu_full"] = caps
with open(os.path.join(out_dir, f"{tag}_ncu_summary.json"), "w") as f:
    json.dump(summary, f, indent=1)

# per-launch DRAM traffic of the GEMM kernel (read by bench.py for roofline.traffic)
tb = []
for d in caps:
    if "gemel_gemm" in d.get("kernel", "") or True:
        try:
            def mb(s):
                v, u = s.split()
                return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            tb.append(mb(d["dram__bytes_read.sum"]) + mb(d["dram__bytes_write.sum"]))
        except Exception:
            pass
if tb and os.environ.get("WRITE_GEMM_TRAFFIC"):
    with open(os.path.join(out_dir, "ncu_gemm_traffic.json"), "w") as f:
        json.dump({"source": f"{tag} ncu --set full capture(s) of gemel_gemm_sm100",
                   "dram_bytes_per_launch": tb if len(tb) > 1 else tb[0],
                   "dram_bytes_per_step_gemm_sum": sum(tb)}, f, indent=1)
print(json.dumps(summary, indent=1)[:3000])
