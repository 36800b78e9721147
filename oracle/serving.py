"""Oracle of the SLA serving loop -- test infrastructure only.

A plain discrete-time (1 ms tick) reference for the serving semantics the library's
event-driven simulator (paper_2201_07705_b200.serving) implements, written from
PAPER.md §3.2 ("a per-frame processing SLA", "skipped ... frames") and
§6 (30 fps feeds, 100 ms SLA), with reading R23:

  * stream s delivers frame k at t = k * 1000 / fps ms (all streams in phase), with
    deadline t + sla;
  * the GPU runs merged steps back to back; a step starting at t0 takes T ms and
    serves every stream with up to B frames: first every queued frame whose deadline
    is before t0 + T is skipped, then the B OLDEST remaining frames of each stream are
    taken (all complete at t0 + T, within their deadlines);
  * a step with no frame left after the skips is not run; the GPU idles (tick by
    tick) while no stream has a frame; a step that would end past the horizon is not
    started; frames still queued at the end are pending (neither processed nor skipped).
Returns per-stream (arrived, processed, skipped, pending).
"""
from __future__ import annotations


def tick_simulate(n_streams, fps, sla_ms, batch, step_ms, duration_ms):
    """step_ms: integer step duration (ms) -- the tick reference only handles whole ms."""
    period = 1000.0 / fps
    queues = [[] for _ in range(n_streams)]          # deadlines (ms) of queued frames, oldest first
    arrived = [0] * n_streams
    processed = [0] * n_streams
    skipped = [0] * n_streams
    next_k = 0                                       # next frame index (same for every stream)
    busy_until = 0
    t = 0
    while t < duration_ms:
        while next_k * period <= t and next_k * period < duration_ms:   # arrivals at this tick
            for s in range(n_streams):
                queues[s].append(next_k * period + sla_ms)
                arrived[s] += 1
            next_k += 1
        # a step starts when the GPU is free, a frame is queued and it ends within the horizon
        # (a step with no frame left after skipping is not run)
        if t >= busy_until and any(queues) and t + step_ms <= duration_ms:
            ran = False
            for s in range(n_streams):
                keep = [d for d in queues[s] if d >= t + step_ms]
                skipped[s] += len(queues[s]) - len(keep)
                take = keep[:batch]
                processed[s] += len(take)
                queues[s] = keep[len(take):]
                ran |= bool(take)
            if ran:
                busy_until = t + step_ms
        t += 1
    pending = [len(q) for q in queues]
    return [(arrived[s], processed[s], skipped[s], pending[s]) for s in range(n_streams)]
