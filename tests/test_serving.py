"""N1: the SLA serving loop.  The
tick-based oracle (oracle.serving) is pinned by closed forms and a hand-traced
timeline; the library's event-driven simulator must equal it exactly on random
instances, and select_batch must be the exhaustive argmax."""
import random

import pytest

from oracle.serving import tick_simulate
from paper_2201_07705_b200.serving import select_batch, simulate


def test_tick_oracle_closed_forms():
    # a step (20 ms) shorter than the frame period (100 ms), SLA 100 ms: every frame is
    # served right after it arrives; conservation arrived = processed + skipped + pending
    r = tick_simulate(3, 10, 100, 1, 20, 1000)
    assert r == [(10, 10, 0, 0)] * 3
    # a step longer than the SLA can never meet a deadline: nothing is processed, and since
    # a step with no frame left is not run, every frame is skipped except the last ones
    r = tick_simulate(2, 10, 100, 4, 150, 1000)
    a, p, s, q = r[0]
    assert p == 0 and a == 10 and s + q == 10 and q <= 2
    # hand trace, 25 fps (period 40 ms), SLA 100 ms, B = 2, step 70 ms, 400 ms horizon:
    #   t=0   queue {f0 dl100}            -> takes f0, busy to 70
    #   t=70  queue {f1 dl140}            -> 140 >= 140: takes f1, busy to 140
    #   t=140 queue {f2 dl180, f3 dl220}  -> 180 < 210: f2 skipped; takes f3, busy to 210
    #   t=210 queue {f4 dl260, f5 dl300}  -> f4 skipped; takes f5, busy to 280
    #   t=280 queue {f6 dl340, f7 dl380}  -> 340 < 350: f6 skipped; takes f7, busy to 350
    #   t=350 queue {f8 dl420}            -> a step would end at 420 > 400: not started
    #   f8, f9 pending: processed 5, skipped 3, pending 2
    assert tick_simulate(1, 25, 100, 2, 70, 400) == [(10, 5, 3, 2)]


def test_event_simulator_equals_tick_oracle():
    rng = random.Random(11)
    for _ in range(300):
        fps = rng.choice([10, 20, 25, 40, 50])
        sla, b, step = rng.choice([50, 100, 150, 200]), rng.choice([1, 2, 3, 4, 8]), rng.randint(1, 150)
        dur = rng.choice([500, 1000, 3000])
        assert simulate(2, fps, sla, b, float(step), dur) == tick_simulate(2, fps, sla, b, step, dur), \
            (fps, sla, b, step, dur)


def test_select_batch_is_the_exhaustive_argmax():
    rng = random.Random(5)
    for _ in range(30):
        base, per = rng.uniform(5, 60), rng.uniform(2, 20)
        steps = {b: base + per * b for b in (1, 2, 4, 8, 16)}
        best, rep = select_batch(steps, 4, 30, 100, duration_ms=5000)
        tput = {b: min(p for _, p, _, _ in simulate(4, 30, 100, b, steps[b], 5000)) for b in steps}
        top = max(tput.values())
        assert tput[best] == top and best == min(b for b in steps if tput[b] == top)
        assert rep[best]["min_fps"] == pytest.approx(top / 5.0)


def test_faster_steps_never_process_fewer_frames():
    """Monotonicity used by the merged-vs-unmerged comparison: a shorter step (merged,
    no weight swap) processes at least as many frames at the same batch."""
    for b in (1, 2, 4, 8):
        prev = None
        for step in (200, 120, 80, 40, 20, 10):
            p = simulate(1, 30, 100, b, float(step), 10_000)[0][1]
            assert prev is None or p >= prev
            prev = p
