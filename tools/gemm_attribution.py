"""Per-layer-class roofline table of the grouped GEMM kernel from a GEMEL_TRACE_DIR
capture (tools/trace_step.py writes plan.json + launch<i>.bin).

Attribution: every CTA (SM) runs its tiles in order; the SM time between the MMA
start of one of its tiles (first k-stage landed) and the MMA start of its next tile
is charged to the first tile (the last tile: until its completion is published).
A problem's SM-time / 148 is its share of the launch; achieved TFLOP/s =
algorithmic FLOPs (2 M N K with the real K) / that share.  Idle SM time (waiting
for dependencies before the first tile, after the last) is reported separately.

    python tools/gemm_attribution.py <trace_dir> [peak_tflops] > table.json
"""
import json
import os
import sys
from collections import defaultdict

import numpy as np


def classify(p):
    k = p.get("kh", 0), p.get("kw", 0)
    kind = "fc" if p.get("linear") else ("stem" if p.get("cols") else f"{k[0]}x{k[1]}s{p.get('sh', 1)}")
    n = p["N"]
    nb = "N<=64" if n <= 64 else "N<=128" if n <= 128 else "N<=256" if n <= 256 else "N>256"
    return f"{kind} {nb}"


def main():
    d = json.load(open(sys.argv[1] + "/plan.json"))
    mp = {}
    mpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(mpath):
        mp = json.load(open(mpath))
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else float(mp.get("bf16_tflops", 1590.0))   # burst, TFLOP/s
    hbm = float(sys.argv[3]) if len(sys.argv) > 3 else float(mp.get("hbm_gbs", 6650.0))        # GB/s
    plan = d["plan"]
    ms_of = [l["ms"] for l in d["launches"]]
    rows = defaultdict(lambda: {"problems": 0, "tiles": 0, "gflop": 0.0, "mb": 0.0, "sm_us": 0.0})
    per_launch = []
    for li, L in enumerate(plan["launches"]):
        if L["kind"] != "gemm" or L.get("stem"):   # the fused first-conv launch is not the grouped kernel
            continue
        try:
            raw = np.fromfile(f"{sys.argv[1]}/launch{li}.bin", dtype=np.uint64).reshape(-1, 16).astype(np.int64)
        except FileNotFoundError:
            continue
        t = raw[:, :8].astype(np.float64) / 1e3          # us
        # a split-K tile parked as a partial never publishes (slot 7 unwritten): its end is
        # its last recorded timestamp
        t[:, 7] = np.where(raw[:, 7] > 0, t[:, 7], np.maximum.reduce([t[:, 3], t[:, 4], t[:, 5], t[:, 6]]))
        cta = raw[:, 8]
        owner = np.empty(len(raw), dtype=np.int64)
        begin = 0
        flops = []
        for pi, p in enumerate(L["problems"]):
            step = L.get("cg", 1) * p.get("msub", 1)   # a tile: msub sub-tiles, or a CTA pair's rows
            mt = -(-(-(-p["M"] // 128)) // step)
            n = mt * -(-p["N"] // p["bn"]) * p.get("ksplit", 1)
            owner[begin:begin + n] = pi
            begin += n
            flops.append(2.0 * p["M"] * p["N"] * p["K"])
        sm_us = np.zeros(len(L["problems"]))
        idle = 0.0
        t_begin, t_end = t[:, 0].min(), t[:, 7].max()
        for c in np.unique(cta):
            idx = np.where(cta == c)[0]
            idx = idx[np.argsort(t[idx, 3])]
            starts = t[idx, 3]
            ends = np.append(starts[1:], t[idx[-1], 7])
            np.add.at(sm_us, owner[idx], (ends - starts) * L.get("cg", 1))   # a pair tile holds 2 SMs
            idle += ((starts[0] - t_begin) + (t_end - t[idx[-1], 7])) * L.get("cg", 1)
        n_sm = 148
        span = t_end - t_begin
        for pi, p in enumerate(L["problems"]):
            r = rows[classify(p)]
            r["problems"] += 1
            r["tiles"] += int((owner == pi).sum())
            r["gflop"] += flops[pi] / 1e9
            r["mb"] += p.get("bytes", 0.0) / 1e6
            r["sm_us"] += sm_us[pi]
        per_launch.append({"launch": li, "problems": len(L["problems"]), "span_us": span,
                           "event_ms": ms_of[li] if li < len(ms_of) else None,
                           "gflop": sum(flops) / 1e9, "tflops": sum(flops) / (span * 1e-6) / 1e12,
                           "idle_sm_frac": idle / (n_sm * span)})
    table = []
    for k, r in sorted(rows.items(), key=lambda kv: -kv[1]["sm_us"]):
        us = r["sm_us"] / 148
        tf = r["gflop"] * 1e9 / (us * 1e-6) / 1e12 if us > 0 else 0.0
        floor_us = max(r["gflop"] * 1e3 / peak, r["mb"] / hbm * 1e3)   # roofline: max(FLOP / peak, bytes / BW)
        table.append({"class": k, "problems": r["problems"], "tiles": r["tiles"], "gflop": round(r["gflop"], 2),
                      "algorithmic_mb": round(r["mb"], 1), "attributed_us": round(us, 1), "tflops": round(tf, 1),
                      "frac_of_tensor_peak": round(tf / peak, 3),
                      "bound": "tensor" if r["gflop"] * 1e3 / peak >= r["mb"] / hbm * 1e3 else "hbm",
                      "roofline_us": round(floor_us, 1), "frac_of_roofline": round(floor_us / us, 3) if us else None})
    json.dump({"peak_tflops": peak, "hbm_gbs": hbm, "note": "per layer class: attributed = SM-time between "
               "consecutive MMA starts / 148; roofline = max(FLOPs / peak, algorithmic bytes / HBM)",
               "by_class": table, "by_launch": per_launch}, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
