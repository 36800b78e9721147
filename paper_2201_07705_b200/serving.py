"""Merge-aware SLA serving loop: frames of every camera stream
arrive at a fixed rate, each must be processed within an SLA of its arrival
("adhering to an SLA (i.e., a per-frame processing deadline)"
"a per-frame processing SLA of 100 ms"), and the GPU runs merged steps back to back.

On B200 a step runs every query of the GPU once over B frames per stream (one graph,
shared layers unioned), so the serving decision is the batch B: the profiler measures
the step time T(B) through the library, `select_batch` picks the B whose simulated
steady state maximises the minimum per-stream throughput ("maximizes the minimum
achieved per-model throughput while adhering to an SLA"), and `serve_live` runs the
real loop against wall-clock arrivals.  Under an HBM weight budget the unmerged
workload streams weights every step (a10) and its T(B) grows; merging removes that
(the paper's frames-skipped result, P:191 / P:431).

Semantics (reading R23): arrivals in phase at t = k * 1000 / fps ms with
deadline t + sla; a step starting at t0 first skips every queued frame whose deadline
is before t0 + T, then takes the B oldest remaining frames of every stream (no frame
left: no step); the GPU idles until a frame is queued; a step that would end past the
horizon is not started.
"""
from __future__ import annotations

import math
import statistics
import time


def simulate(n_streams, fps, sla_ms, batch, step_ms, duration_ms):
    """Event-driven steady-state simulation.  Returns per-stream (arrived, processed,
    skipped, pending) -- streams are in phase, so every stream has the same counts."""
    period = 1000.0 / fps
    n_arrivals = math.ceil(duration_ms / period)          # frames k with k * period < duration
    q = []                                                # deadlines of queued frames (one stream)
    k_next = 0
    t_free = 0.0
    processed = skipped = 0
    while True:
        if not q:
            if k_next >= n_arrivals:
                break
            t0 = max(t_free, k_next * period)
        else:
            t0 = t_free
        if t0 + step_ms > duration_ms:
            break
        while k_next < n_arrivals and k_next * period <= t0:
            q.append(k_next * period + sla_ms)
            k_next += 1
        keep = [d for d in q if d >= t0 + step_ms]
        skipped += len(q) - len(keep)
        take = min(batch, len(keep))
        processed += take
        q = keep[take:]
        if take:                                          # a step with nothing left to run is not run
            t_free = t0 + step_ms
    pending = n_arrivals - processed - skipped
    return [(n_arrivals, processed, skipped, pending)] * n_streams


def select_batch(step_ms_of, n_streams, fps, sla_ms, duration_ms=60_000):
    """The batch maximising the minimum per-stream throughput (processed frames per
    second) in the simulated steady state; ties -> the smaller batch (lower latency).
    step_ms_of: {B: measured step ms}.  Returns (B, {B: report})."""
    reports = {}
    best = None
    for b in sorted(step_ms_of):
        r = simulate(n_streams, fps, sla_ms, b, step_ms_of[b], duration_ms)
        tput = min(p for _, p, _, _ in r) / (duration_ms / 1000.0)
        reports[b] = {"step_ms": step_ms_of[b], "min_fps": tput, "per_stream": r[0]}
        if best is None or tput > reports[best]["min_fps"] + 1e-9:
            best = b
    return best, reports


def profile_step_ms(wl, frames, outs, steps=20, warmup=3):
    """Median device time of one merged step (CUDA events on the library's stream)."""
    import torch
    for _ in range(warmup):
        wl.infer(frames, outs)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(wl.stream)
        wl.infer(frames, outs)
        b.record(wl.stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def serve_live(wl, host_frames, host_outs, fps, sla_ms, duration_s, step_estimate_ms):
    """The serving loop run for real: frames 'arrive' on the wall clock, each step
    copies the chosen frames from pinned host memory, runs the merged step and reads
    the results back (gemel_infer with host buffers); a frame counts as processed when
    its step completed by its deadline.  Same policy as `simulate`, with the expected
    step time for the skip decision.  Returns per-stream-equal counts and timings."""
    import torch
    batch = next(iter(host_frames.values())).shape[0]
    period = 1000.0 / fps
    n_arrivals = math.ceil(duration_s * 1000.0 / period)
    q = []
    k_next = 0
    processed = skipped = late = steps = 0
    step_times = []
    t_start = time.perf_counter()

    def now_ms():
        return (time.perf_counter() - t_start) * 1000.0
    while True:
        t0 = now_ms()
        while k_next < n_arrivals and k_next * period <= t0:
            q.append(k_next * period + sla_ms)
            k_next += 1
        if not q:
            if k_next >= n_arrivals:
                break
            time.sleep(max(0.0, (k_next * period - t0) / 1000.0))
            continue
        if t0 + step_estimate_ms > duration_s * 1000.0:
            break
        keep = [d for d in q if d >= t0 + step_estimate_ms]
        skipped += len(q) - len(keep)
        take = keep[:batch]
        q = keep[len(take):]
        if not take:
            continue
        wl.infer(host_frames, host_outs, on_host=True)
        torch.cuda.current_stream().synchronize()
        wl.stream.synchronize()
        t1 = now_ms()
        step_times.append(t1 - t0)
        steps += 1
        ok = sum(1 for d in take if d >= t1)
        processed += ok
        late += len(take) - ok
    pending = n_arrivals - processed - skipped - late
    return {"arrived": n_arrivals, "processed": processed, "skipped": skipped + late, "late": late,
            "pending": pending, "steps": steps,
            "step_ms_median": statistics.median(step_times) if step_times else None}


class HotSwap:
    """Non-blocking merge-configuration hot-swap (a
    new merged model version is built off the serving path and swapped in): `stage`
    builds the next workload (registration, merge, plan, bind -- everything but the
    steps) on a background thread while the current one keeps serving; `current()`
    returns the workload for the next step and switches at a step boundary once the
    staged one is ready (the old one is closed after its last step completed)."""

    def __init__(self, wl):
        import threading
        self._wl = wl
        self._next = None
        self._err = None
        self._lock = threading.Lock()
        self._thread = None
        self.switches = 0

    def stage(self, build):
        import threading

        def run():
            try:
                nxt = build()
                with self._lock:
                    self._next = nxt
            except Exception as e:   # surfaced by current()
                with self._lock:
                    self._err = e
        self._thread = threading.Thread(target=run, daemon=True)
        self._thread.start()

    def current(self):
        with self._lock:
            if self._err is not None:
                raise self._err
            nxt, self._next = self._next, None
        if nxt is not None:
            self._wl.stream.synchronize()     # the old configuration's last step is done
            self._wl.close()
            self._wl = nxt
            self.switches += 1
        return self._wl

    def wait_staged(self):
        if self._thread is not None:
            self._thread.join()
