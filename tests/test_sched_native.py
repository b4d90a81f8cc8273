"""libfae's scheduler (fae_sched_*, host-only C++, NEXT-3) against the
scheduler oracle (oracle/sched.py, itself pinned by tests/test_sched_oracle.py)
— CPU only: the scheduler launches nothing."""
import random

import pytest

from oracle import sched as osched


def fae():
    import paper_2103_00686_b200 as m
    return m


def _run(m, nc, nh, r0, u, losses, epochs=1):
    a = m.Scheduler(nc, nh, r0, u)
    b = osched.Scheduler(nc, nh, r0, u)
    trace = []
    li = 0
    for ep in range(epochs):
        if ep:
            a.new_epoch()
            b.new_epoch()
        while True:
            pa, pb = a.next_phase(), b.next_phase()
            if pb is None:
                assert pa is None
                break
            assert pa[:3] == pb, (pa, pb)
            assert pa[3] == b.pending_swap()
            trace.append(pa)
            if pa[3]:
                v = losses[li % len(losses)]
                li += 1
                a.record_swap(v, 4096, 8)
                b.record_swap(v, 4096, 8)
                assert a.rate == b.r
    assert a.swaps == b.swaps and a.s.sync_bytes == b.sync_bytes and a.s.sync_events == b.sync_events
    return trace


def test_native_equals_oracle_random():
    m = fae()
    rng = random.Random(11)
    for _ in range(300):
        nc, nh = rng.randint(0, 80), rng.randint(0, 80)
        r0 = rng.choice([1.0, 2.0, 7.5, 25.0, 50.0, 100.0])
        u = rng.choice([1, 2, 4, 6])
        walk, v = [], 0.7
        for _ in range(64):
            v += rng.choice([-0.02, -0.01, 0.0, 0.01, 0.03])
            walk.append(v)
        _run(m, nc, nh, r0, u, walk, epochs=rng.choice([1, 2, 3]))


def test_native_golden_plans():
    m = fae()
    assert [(k, c) for k, _, c, _ in _run(m, 100, 100, 50, 4, [0.5])] == \
        [("cold", 50), ("hot", 50), ("cold", 50), ("hot", 50)]
    assert [(k, c) for k, _, c, _ in _run(m, 10, 4, 1, 4, [0.5])] == \
        [("cold", 1), ("hot", 1)] * 4 + [("cold", 6)]


def test_native_trajectory():
    m = fae()
    s = m.Scheduler(10_000, 10_000, 50.0)
    got = []
    for v in (0.5, 0.52, 0.51, 0.50, 0.49, 0.48, 0.47):
        s.record_swap(v)
        got.append(s.rate)
    assert got == [50, 25, 25, 25, 25, 50, 100]


def test_native_bad_arguments():
    m = fae()
    with pytest.raises(m.FaeError):
        m.Scheduler(1, 1, 0.5)
    with pytest.raises(m.FaeError):
        m.Scheduler(1, 1, 50, u=0)
    s = m.Scheduler(1, 1, 50)
    with pytest.raises(m.FaeError):
        s.record_swap(float("nan"))
