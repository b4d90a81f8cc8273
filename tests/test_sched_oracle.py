"""Pins of the scheduler oracle (oracle/sched.py) against what PAPER.md §4.3
(Eq. 5) and SPEC.md's worked examples fix — CPU only."""
import os
import random

import pytest

from oracle import sched

GOLD = os.path.join(os.path.dirname(__file__), "golden", "scheduler_examples.txt")


def _gold(kind):
    for ln in open(GOLD):
        ln = ln.strip()
        if ln and not ln.startswith("#") and ln.startswith(kind + " "):
            yield [p.strip() for p in ln[len(kind) + 1:].split("|")]


def test_next_rate_examples():
    n = 0
    for r, losses, want in _gold("rate"):
        got = sched.next_rate(float(r), [float(v) for v in losses.split(",")], 4)
        assert got == float(want), (r, losses, got)
        n += 1
    assert n == 5


def test_rate_trajectory_example():
    for r, losses, want in _gold("traj"):
        s = sched.Scheduler(10_000, 10_000, float(r))
        got = []
        for v in losses.split(","):
            s.record_swap(float(v))
            got.append(s.r)
        assert got == [float(w) for w in want.split(",")]


def test_fixed_plans():
    for head, want in _gold("plan"):
        nc, nh, r = head.split()
        got = sched.plan_fixed(int(nc), int(nh), float(r))
        assert [f"{k[0].upper()}{c}" for k, c in got] == want.split(","), (head, got)


def test_invariants_random_losses():
    """Conservation (every batch once, in order per kind), cold first, rate
    bounds [1, 100], rate changes only at swaps, u-window doubling, swaps
    bounded by the R(1) and R(100) plans."""
    rng = random.Random(5)
    for trial in range(200):
        nc, nh = rng.randint(0, 60), rng.randint(0, 60)
        r0 = rng.choice([1, 3, 12.5, 25, 50, 100])
        s = sched.Scheduler(nc, nh, r0)
        seen = {"cold": [], "hot": []}
        first = None
        loss = 1.0
        while True:
            p = s.next_phase()
            if p is None:
                break
            k, f, c = p
            first = first or k
            assert c >= 1
            seen[k].extend(range(f, f + c))
            if s.pending_swap():
                loss += rng.uniform(-0.05, 0.04)
                r_before = s.r
                s.record_swap(loss, hot_bytes=1000, n_devices=2)
                assert 1.0 <= s.r <= 100.0
                assert s.r in (r_before, max(r_before / 2, 1.0), min(r_before * 2, 100.0))
        assert seen["cold"] == list(range(nc)) and seen["hot"] == list(range(nh))
        if nc > 0:
            assert first == "cold"
        assert s.sync_events == 2 * s.swaps and s.sync_bytes == 2000 * s.swaps
        lo = 1 if (nc and nh) else 0
        hi = max(0, 2 * min(nc, nh) - (0 if nc > nh else 1)) if (nc and nh) else 0
        assert lo <= s.swaps <= max(hi, lo)


def test_halving_and_doubling_reach_bounds():
    s = sched.Scheduler(1000, 1000, 50.0)
    v = 1.0
    for _ in range(10):           # every loss rises: 50 -> 25 -> ... -> 1
        v += 0.1
        s.record_swap(v)
    assert s.r == 1.0
    for _ in range(40):           # every loss falls: doubles every swap once u = 4 decreases
        v -= 0.01
        s.record_swap(v)
    assert s.r == 100.0


def test_bad_arguments():
    with pytest.raises(ValueError):
        sched.Scheduler(1, 1, 0.5)
    with pytest.raises(ValueError):
        sched.Scheduler(1, 1, 50, u=0)
