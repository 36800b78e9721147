#!/usr/bin/env python
"""Benchmark: merged multi-model inference throughput (frames/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--cfg 4] [--merge cross|full|none]
    python bench.py --impl reference ...      # the CPU fp64 oracle arm

Default workload: cfg4 = 4x YOLOv3 + 4x Faster R-CNN R50-FPN at 608x608, B=4
frames per stream (8 streams, 32 frames per step) -- the largest BASELINE.json
configuration that fits one GPU (configs[3]; the metric names no config, so the
N=1 line takes the largest single-GPU one; cfg5 is the 8-GPU sharded mix).
Architecturally identical layers are merged across models ("cross": the k-th
appearance of a signature in every model forms one group).
A step = one frame batch per stream through every model (SURVEY.md §8(a)
a6-a11).  Timing: W warm-up steps, then K steps, each bracketed by CUDA events on
the library's stream with a 256 MiB L2 flush between steps (outside the events);
ms_per_step = the median step, the mean is reported too.

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (127.0.0.1).  One process per GPU; each rank
runs its own copy of the workload on its own streams (weak scaling, no data-path
collective); merged weights are broadcast from rank 0 once (NCCL) and each step's
result slab is gathered to rank 0 on a comm stream that overlaps the next step
(SURVEY.md §8(e)).  `--shard` splits one config's queries over the ranks instead.

Synthetic seeded frames and random-init weights (workloads/synth.py).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import configs, synth, zoo  # noqa: E402

FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(FALLBACK_PEAKS)
    d["_source"] = "fallback (B200_PROFILING.md)"
    return d


def query_costs(cfg):
    """Algorithmic conv+linear FLOPs per step of every query of a config, from the
    library's host-side planner (dry plan, no GPU): the bin-packing weights of
    --shard."""
    from paper_2201_07705_b200 import gemel as G
    cache, costs = {}, []
    for name, sid in cfg["queries"]:
        r = configs.stream_res(cfg, sid)
        if (name, r) not in cache:
            layers = zoo.build(name)
            ctx = G.gemel_create(flags=G.FLAG_DRY_PLAN)
            try:
                G.gemel_register_model(ctx, layers, synth.params(layers, 0, 0), 0, r, r)
                cache[(name, r)] = G.gemel_plan(ctx, [cfg["batch"]])["gemm_flops_per_step"]
            finally:
                G.gemel_destroy(ctx)
        costs.append(cache[(name, r)])
    return costs


def build_queries(cfg_id, rank, only=None):
    """Queries of a config (all of them, or the indices in `only` for --shard)."""
    cfg = configs.CONFIGS[cfg_id]
    queries, models, params = [], [], []
    for q, (name, sid) in enumerate(cfg["queries"]):
        if only is not None and q not in only:
            continue
        layers = zoo.build(name)
        p = synth.params(layers, *configs.weight_key(cfg_id, q))   # same weights on every rank
        queries.append((layers, p, sid))
        models.append(layers)
        params.append(p)
    frames = {sid: synth.frames(cfg_id, sid + 1000 * rank, cfg["batch"], configs.stream_res(cfg, sid),
                                configs.stream_res(cfg, sid))
              for _, sid in [(None, s) for _, _, s in queries]}
    return cfg, queries, models, params, frames, len(queries)


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: an NVML thread
    polling every 2 ms (the timed region of a short run lasts only tens of ms), with
    nvidia-smi as the fallback when NVML is unavailable."""

    # NVML clocks-event-reason bits
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = None
        self._thread = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            getr = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self.mx.append(float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)))
        except Exception:
            return self
        self._stop = threading.Event()

        def poll():
            while not self._stop.is_set():
                try:
                    self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    r = getr(h)
                    for n, bit in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(n)
                except Exception:
                    pass
                self._stop.wait(0.002)

        self._thread = threading.Thread(target=poll, daemon=True)
        self._thread.start()
        return self

    def __exit__(self, *a):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=5)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "nvml unavailable"}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx), "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml, 2 ms polling during the timed region"}


def host_cpu():
    """Host CPU model name and the threads the oracle's BLAS uses."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    return model, cores


def oracle_sample_queries(models, names):
    """The bounded CPU sample: one frame of the first query of every distinct
    architecture (cfg4: one YOLOv3 + one Faster R-CNN frame, ~20 s of fp64 NumPy)."""
    seen, picks = set(), []
    for q, n in enumerate(names):
        if n not in seen:
            seen.add(n)
            picks.append(q)
    return picks


def cpu_oracle_sample(models, params, merge_cfg, frames, names, sids):
    """Oracle (NumPy fp64, as it stands) on a bounded sample of the same workload:
    1 frame of one query of every distinct architecture, merged weights."""
    from oracle import merge as om
    from oracle import model as omodel
    model_name, cores = host_cpu()
    mp = om.merged_params(models, params, merge_cfg) if merge_cfg else params
    picks = oracle_sample_queries(models, names)
    t0 = time.perf_counter()
    for q in picks:
        omodel.run(models[q], mp[q], frames[sids[q]][:1])
    dt = time.perf_counter() - t0
    return {"value": len(picks) / dt, "unit": "frames/s", "cores": cores, "cpu": model_name, "kind": "oracle",
            "sample": f"1 frame of each of {len(picks)} distinct architectures "
                      f"({', '.join(names[q] for q in picks)}; {dt:.1f} s of fp64 NumPy)"}


def registered_weight_bytes(models):
    """bf16 bytes of every registered param layer (the budget's 100%)."""
    n = 0
    for layers in models:
        for l in layers:
            if l["op"] == "conv":
                n += l["cout"] * (l["cin"] // l["groups"]) * l["k"][0] * l["k"][1] + (l["cout"] if l["bias"] else 0)
            elif l["op"] == "linear":
                n += l["fout"] * l["fin"] + (l["fout"] if l["bias"] else 0)
            elif l["op"] == "bn":
                n += 4 * l["c"]
    return 2 * n


def run_reference(args):
    """The reference arm: the oracle as it stands on the host cores, on this arm's
    config/metric.  Each step = one frame of one query (queries in rotation), a
    bounded sample of the workload; rank 0 only (other ranks exit without work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, queries, models, params, frames, nq = build_queries(args.cfg, 0)
    from oracle import merge as om
    from oracle import model as omodel
    groups = om.find_shareable(models)
    cfgm = (om.full_merge(groups) if args.merge == "full" else
            om.cross_model_groups(groups) if args.merge == "cross" else [])
    mp = om.merged_params(models, params, cfgm) if cfgm else params
    sids = [sid for _, _, sid in queries]
    names = [n for n, _ in cfg["queries"]]
    model_name, cores = host_cpu()
    # warm-up: the oracle has no device state to warm; W steps would only lengthen the
    # run (a 608x608 frame is ~10 s of fp64), so they are not executed
    times = []
    for k in range(args.steps):
        q = k % nq
        t0 = time.perf_counter()
        omodel.run(models[q], mp[q], frames[sids[q]][:1])
        times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.median(times)
    fps = 1.0 / (sum(times) / len(times))
    sample = f"1 frame of one query per step, queries in rotation ({args.steps} steps, {sum(times):.1f} s)"
    line = {"impl": "reference", "metric": METRIC, "value": fps,
            "unit": "frames/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "ms_per_step_median": ms,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uint8 frames, random-init weights)",
            "config": config_dict(cfg, args, nq, 1, None, 0),
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "cpu": model_name, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


METRIC = "frames/s across all streams (merged workload)"


def config_dict(cfg, args, nq, world, part, budget):
    return {"workload": cfg["name"], "models": [q[0] for q in cfg["queries"]], "streams_per_gpu": nq,
            "batch_per_stream": cfg["batch"], "res": cfg["res"], "res_of": cfg.get("res_of"),
            "frames_per_step_per_gpu": cfg["batch"] * nq, "merge": args.merge,
            "parallelism": (f"{world}-way query partition (bin-packed by FLOPs, sharers co-located)"
                            if args.shard else f"dp{world} (independent streams per GPU)"),
            "partition": part, "weight_budget_bytes": budget,
            "l2": "flushed between timed steps (256 MiB write outside the events)",
            "weight_source": getattr(args, "weight_source", "host")}


def pcie_peak():
    """Measured pinned host -> device bandwidth (MEASURED_PEAKS.json if it carries one,
    else the committed tools/h2d_peak.py measurement)."""
    peaks = load_peaks()
    if "h2d_gbs" in peaks:
        return peaks["h2d_gbs"], peaks["_source"]
    p = os.path.join(ROOT, "profiles", "r2_h2d_peak.json")
    try:
        return json.load(open(p))["h2d_pinned_gbs"], "measured (profiles/r2_h2d_peak.json, tools/h2d_peak.py)"
    except Exception:
        return None, None


def measured_traffic(workload, merge):
    """DRAM bytes per step of the grouped-GEMM launches from the committed ncu capture
    of this workload (profiles/ncu_traffic.json, tools/ncu_traffic.py), or None."""
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(tp))
        e = d.get(f"{workload}:{merge}")
        return (e["gemm_dram_bytes_per_step"], e) if e else (None, None)
    except Exception:
        return None, None


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2201_07705_b200.dist import ResultGather, broadcast_weights, partition_queries
    from paper_2201_07705_b200.engine import MergedWorkload

    part = None
    if args.shard:   # strong scaling: this config's queries bin-packed over the ranks
        cfg0 = configs.CONFIGS[args.cfg]
        part = partition_queries(query_costs(cfg0), [n for n, _ in cfg0["queries"]], world)
        if not part[rank]:
            raise SystemExit(f"--shard: rank {rank} received no query ({len(cfg0['queries'])} queries, {world} ranks)")
    cfg, queries, models, params, frames_np, nq = build_queries(args.cfg, 0 if args.shard else rank,
                                                                part[rank] if part else None)
    budget = int(args.budget_frac * registered_weight_bytes(models)) if args.budget_frac > 0 else 0
    res = {sid: (configs.stream_res(cfg, sid),) * 2 for _, sid in cfg["queries"]}
    src_dev = args.source_device
    if args.weight_source == "peer" and src_dev is None:
        src_dev = (local + 1) % torch.cuda.device_count()
    wl = MergedWorkload(queries, res, cfg["batch"], merge=args.merge, weight_budget=budget,
                        weight_source=args.weight_source, source_device=src_dev)
    bcast_ms = None
    if world > 1:
        # place merged weights once per GPU from rank 0 (NCCL over NVLink).  With --shard the
        # ranks hold different query sets, so each rank's arena is broadcast from the rank
        # that built it only when the arenas match; otherwise every rank keeps its own upload.
        t0 = time.perf_counter()
        if not args.shard:
            broadcast_weights(wl.w_arena, src=0)
        torch.cuda.synchronize()
        bcast_ms = 1e3 * (time.perf_counter() - t0)
    frames = {s: torch.from_numpy(f).cuda() for s, f in frames_np.items()}
    outs = wl.alloc_outputs()
    fps_step = cfg["batch"] * nq                       # frames this rank processes per step
    total_frames = cfg["batch"] * len(cfg["queries"]) if args.shard else world * fps_step
    gather = None
    if world > 1:
        n_out = torch.tensor([sum(o.numel() for o in outs.values())], device="cuda")
        dist.all_reduce(n_out, op=dist.ReduceOp.MAX)
        gather = ResultGather(outs, rank, world, max_numel=int(n_out.item()), compute_stream=wl.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = wl.stream

    def step():
        wl.infer(frames, outs)
        if gather is not None:        # per-step result gather to rank 0 (NCCL, comm stream)
            gather(outs)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            ev[k][0].record(st)
            step()
            ev[k][1].record(st)
            with torch.cuda.stream(st):
                flush.fill_(k & 0xFF)        # L2 flush between timed steps (outside the events)
        torch.cuda.synchronize()
    if world > 1:
        if gather is not None:
            gather.wait()
        dist.barrier()
    per_step = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([statistics.median(per_step), sum(per_step) / len(per_step)], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_med, ms_mean = float(t[0].item()), float(t[1].item())

    # ---- end to end through the public API with host buffers (H2D + D2H in the region)
    hframes = {s: torch.from_numpy(f).pin_memory() for s, f in frames_np.items()}
    houts = wl.alloc_outputs(on_host=True)
    for _ in range(3):
        wl.infer(hframes, houts, on_host=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    e0.record(st)
    for _ in range(args.steps):
        wl.infer(hframes, houts, on_host=True)   # H2D frames, step, D2H logits (pinned host)
    e1.record(st)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([e2e_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    h2d = sum(f.numel() for f in hframes.values())
    d2h = sum(o.numel() * 4 for o in houts.values())

    # ---- roofline of the dominant kernel (grouped implicit-GEMM): per-launch CUDA events
    # on the library's stream in profiling mode (same launches as the graph, no capture)
    wl.set_profiling(True)
    prof_runs = []
    for _ in range(5):
        wl.infer(frames, outs)
        torch.cuda.synchronize()
        prof_runs.append(wl.launch_list())
    wl.set_profiling(False)
    prof = prof_runs[-1]
    n_l = len(prof)
    for i in range(n_l):   # per-launch median over the profiled steps
        prof[i]["ms"] = statistics.median(r[i]["ms"] for r in prof_runs[1:])
    gemm = [l for l in prof if l["kind"] == "gemm"]
    g_ms = sum(l["ms"] for l in gemm)
    g_flops = sum(l["flops"] for l in gemm)
    all_ms = sum(l["ms"] for l in prof)
    peaks = load_peaks()
    achieved = g_flops / (g_ms * 1e-3) / 1e12 if g_ms > 0 else 0.0
    # the GEMM launches are timed alone (ms-scale launches in a ~10 ms step): burst peak
    peak = peaks["bf16_tflops"]
    traffic, traffic_src = measured_traffic(cfg["name"], args.merge)
    by_kind = {}
    for l in prof:
        k = by_kind.setdefault(l["kind"], {"launches": 0, "ms": 0.0, "gflop": 0.0, "mb": 0.0})
        k["launches"] += 1
        k["ms"] += l["ms"]
        k["gflop"] += l["flops"] / 1e9
        k["mb"] += l["bytes"] / 1e6

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC,
            "value": total_frames / (ms_med * 1e-3),
            "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": ms_med, "ms_per_step_mean": ms_mean, "timing": "median of per-step CUDA events "
            "(max over ranks); value = frames per step (all ranks) / median step",
            "higher_is_better": True, "scaling": "strong" if args.shard else "weak",
            "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (seeded uint8 frames, random-init weights)",
            "config": config_dict(cfg, args, nq, world, part, budget),
            "merge": {"bytes_saved": wl.bytes_saved, "weight_gb_saved": wl.bytes_saved / 1e9,
                      "unmerged_weight_bytes": wl.plan["unmerged_weight_bytes"],
                      "unique_weight_bytes": wl.plan["unique_weight_bytes"],
                      "reduction": wl.bytes_saved / max(wl.plan["unmerged_weight_bytes"], 1),
                      "union_problems": wl.plan["n_union_problems"], "gemm_problems": wl.plan["n_gemm_problems"]},
            "swap": {"bytes_per_step": wl.plan["swap_bytes_per_step"], "tensors": wl.plan["n_swapped"],
                     "pinned_bytes": wl.plan["pinned_weight_bytes"], "ring_bytes": wl.plan["swap_ring_bytes"]},
            "e2e": {"value": total_frames / (e2e_ms * 1e-3), "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": wl.plan["n_launches"] * args.steps,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "gemel_gemm_sm100 (all grouped GEMM launches of a step)",
                         "peak_source": peaks["_source"] + " bf16_tflops (burst: launches timed alone)",
                         "traffic_source": traffic_src,
                         "gemm_share_of_step": g_ms / all_ms if all_ms else None,
                         "gemm_ms_per_step": g_ms, "gemm_tflop_per_step": g_flops / 1e12,
                         "step_tflops": wl.plan["gemm_flops_per_step"] / (ms_med * 1e-3) / 1e12,
                         "by_kind": by_kind},
            "clocks": clocks,
        }
        if wl.plan["swap_bytes_per_step"] > 0:   # weights streamed every step: the copy term of the roofline
            if args.weight_source == "peer" and src_dev != local:
                bound, h2d, h2d_src = "nvlink", 770.0, "B200_PROFILING.md measured peer copy per direction"
            elif args.weight_source == "peer":   # paged within HBM: a copy reads and writes every byte
                bound, h2d, h2d_src = "hbm", peaks["hbm_gbs"] / 2, peaks["_source"] + " hbm_gbs / 2 (copy)"
            else:
                bound, (h2d, h2d_src) = "pcie", pcie_peak()
            floor_ms = wl.plan["swap_bytes_per_step"] / (h2d * 1e9) * 1e3 if h2d else None
            line["swap_roofline"] = {"bound": bound, "bytes_per_step": wl.plan["swap_bytes_per_step"],
                                     "peak_gbs": h2d, "peak_source": h2d_src, "floor_ms": floor_ms,
                                     "achieved_gbs": wl.plan["swap_bytes_per_step"] / (ms_med * 1e-3) / 1e9,
                                     "frac": floor_ms / ms_med if floor_ms else None}
        if bcast_ms is not None:
            line["weight_broadcast_ms"] = bcast_ms
        if world == 1 and not args.no_cpu:
            names = [n for n, _ in cfg["queries"]]
            sids = [sid for _, _, sid in queries]
            line["cpu_baseline"] = cpu_oracle_sample(models, params, oracle_merge_config(models, args.merge),
                                                     frames_np, names, sids)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    wl.close()
    return 0


def oracle_merge_config(models, merge):
    """The oracle's own merge configuration for the cpu_baseline leg."""
    from oracle import merge as om
    groups = om.find_shareable(models)
    return (om.full_merge(groups) if merge == "full" else
            om.cross_model_groups(groups) if merge == "cross" else [])


def relaunch_distributed(args_list, n):
    """`--gpus N` outside torchrun: re-launch this script with N ranks on 127.0.0.1."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + args_list
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--cfg", type=int, default=4)
    ap.add_argument("--merge", default="cross", choices=["cross", "full", "none"],
                    help="cross: cross-model groups (SURVEY.md §8 benchmark reading); full: every group in full")
    ap.add_argument("--impl", default="gemel", choices=["gemel", "reference"])
    ap.add_argument("--budget-frac", type=float, default=0.0,
                    help="HBM weight budget as a fraction of the registered (unmerged) weight bytes; 0 = unlimited")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline oracle leg")
    ap.add_argument("--weight-source", default="host", choices=["host", "peer"],
                    help="page weights above the budget from pinned host memory or a peer GPU's HBM (N4)")
    ap.add_argument("--source-device", type=int, default=None,
                    help="GPU holding the paged weights for --weight-source peer (default: the next GPU, "
                         "or this one on a 1-GPU box)")
    ap.add_argument("--shard", action="store_true",
                    help="strong scaling: split the config's queries over the ranks (bin packing, SURVEY.md §8(e)) "
                         "instead of one copy of the workload per rank")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(sys.argv[1:], args.gpus)
    if args.impl == "reference" and args.steps == ap.get_default("steps"):
        args.steps = 20   # bounded CPU sample: ~10 s per 608x608 frame of fp64 NumPy
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
