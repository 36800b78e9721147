"""N1 measurement: the merge-aware SLA serving loop on one B200.

For a config under an HBM weight budget (default cfg5, 50% of the unmerged weights,
the paper's "50%" memory setting P:126), unmerged and cross-merged: profile the step
time T(B) through the library for B in {1, 2, 4, 8}, pick the batch maximising the
minimum per-stream throughput under the SLA (30 fps, 100 ms) in a 60 s
simulated steady state, then run the real serving loop for a few seconds against
wall-clock arrivals with host frames.  Prints one JSON object.

    python tools/serve_sla.py [--cfg 5] [--budget-frac 0.5] [--live-s 5]
"""
import argparse
import gc
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_07705_b200 import serving  # noqa: E402
from paper_2201_07705_b200.engine import MergedWorkload  # noqa: E402
from workloads import configs, synth, zoo  # noqa: E402


def registered_bytes(models):
    n = 0
    for layers in models:
        for l in layers:
            if l["op"] == "conv" and "tie" not in l:
                n += l["cout"] * (l["cin"] // l["groups"]) * l["k"][0] * l["k"][1] + (l["cout"] if l["bias"] else 0)
            elif l["op"] == "linear":
                n += l["fout"] * l["fin"] + (l["fout"] if l["bias"] else 0)
            elif l["op"] == "bn":
                n += 4 * l["c"]
    return 2 * n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--budget-frac", type=float, default=0.5)
    ap.add_argument("--budget-min", action="store_true",
                    help="the paper's 'min' memory setting: the largest single model's weights (P:126)")
    ap.add_argument("--fps", type=float, default=30.0)
    ap.add_argument("--sla-ms", type=float, default=100.0)
    ap.add_argument("--batches", default="1,2,4,8")
    ap.add_argument("--live-s", type=float, default=5.0)
    args = ap.parse_args()
    cfg = configs.CONFIGS[args.cfg]
    names = [n for n, _ in cfg["queries"]]
    sids = [s for _, s in cfg["queries"]]
    models = [zoo.build(n) for n in names]
    params = [synth.params(m, *configs.weight_key(args.cfg, q)) for q, m in enumerate(models)]
    res = {s: (configs.stream_res(cfg, s),) * 2 for s in sids}
    if args.budget_min:
        # the paper's "min" setting: memory for the largest model; raised in 10%
        # steps until the unmerged workload can double-buffer its largest streamed tensor
        from paper_2201_07705_b200 import gemel as G
        budget = max(registered_bytes([m]) for m in models)
        while True:
            ctx = G.gemel_create(flags=G.FLAG_DRY_PLAN, weight_budget_bytes=budget)
            try:
                for q, m in enumerate(models):
                    G.gemel_register_model(ctx, m, params[q], sids[q], *res[sids[q]])
                G.gemel_plan(ctx, [1] * (max(sids) + 1))
                break
            except G.GemelError as e:
                if e.code != G.E_NOMEM:
                    raise
                budget = int(budget * 1.1)
            finally:
                G.gemel_destroy(ctx)
    else:
        budget = int(args.budget_frac * registered_bytes(models))
    out = {"workload": cfg["name"], "streams": len(sids), "fps": args.fps, "sla_ms": args.sla_ms,
           "weight_budget_bytes": budget, "budget": "min (largest model)" if args.budget_min else args.budget_frac,
           "runs": {}}
    for merge in ("none", "cross"):
        steps = {}
        swap = {}
        for b in [int(x) for x in args.batches.split(",")]:
            wl = MergedWorkload([(m, p, s) for m, p, s in zip(models, params, sids)], res, b, merge=merge,
                                weight_budget=budget)
            fr = {s: torch.from_numpy(synth.frames(args.cfg, s, b, *res[s])).cuda() for s in sids}
            outs = wl.alloc_outputs()
            steps[b] = serving.profile_step_ms(wl, fr, outs)
            swap[b] = wl.plan["swap_bytes_per_step"]
            wl.close()
            del wl, fr, outs
            gc.collect()
            torch.cuda.empty_cache()
        best, rep = serving.select_batch(steps, len(sids), args.fps, args.sla_ms)
        wl = MergedWorkload([(m, p, s) for m, p, s in zip(models, params, sids)], res, best, merge=merge,
                            weight_budget=budget)
        hfr = {s: torch.from_numpy(synth.frames(args.cfg, s, best, *res[s])).pin_memory() for s in sids}
        houts = wl.alloc_outputs(on_host=True)
        for _ in range(3):
            wl.infer(hfr, houts, on_host=True)
        torch.cuda.synchronize()
        live = serving.serve_live(wl, hfr, houts, args.fps, args.sla_ms, args.live_s, steps[best])
        out["runs"][merge] = {"step_ms": steps, "swap_bytes_per_step": swap, "batch": best,
                              "simulated_60s": rep, "live": live, "bytes_saved": wl.bytes_saved}
        wl.close()
        del wl
        gc.collect()
        torch.cuda.empty_cache()
    u, m = out["runs"]["none"], out["runs"]["cross"]
    out["summary"] = {
        "sim_processed_fraction": {k: v["simulated_60s"][v["batch"]]["per_stream"][1] /
                                   v["simulated_60s"][v["batch"]]["per_stream"][0] for k, v in out["runs"].items()},
        "live_processed_fraction": {k: v["live"]["processed"] / v["live"]["arrived"] for k, v in out["runs"].items()},
        "live_more_frames_merged": m["live"]["processed"] / max(u["live"]["processed"], 1) - 1.0}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
