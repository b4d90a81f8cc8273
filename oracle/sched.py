"""CPU ORACLE of the hot/cold scheduler (Eq. 5) — TEST INFRASTRUCTURE ONLY.

Only tests/ (and bench.py's oracle legs) may import this module; the product
path (paper_2103_00686_b200, libfae's fae_sched_*) never does, and nothing
here comes from it.  Plain Python, written step by step from PAPER.md §4.3
("Communication Overheads" and Eq. 5 `eqn:scheduler`),
with SPEC.md's reading of the garbled parts — DESIGN.md R28-R31:

  * R(r): a phase issues ceil(r% of the kind's ORIGINAL per-epoch batch
    count) batches of one kind before swapping ("R(100) implies
    that 100% of the mini-batches of cold inputs will be completed before
    the first hot mini-batches is issued. A rate of (R(1)) implies hot and
    cold are shuffled after every mini-batch").
  * cold first ("The scheduler always begins with training on cold
    inputs"), start at R(50); when one kind is drained the rest of
    the other kind is issued as one phase (no swap is possible).
  * Eq. 5 at each swap i with the post-swap test loss Test_L(i):
      Test_L(i) > Test_L(i-1)                         -> r = max(r/2, 1)
      else the last u losses strictly decreased      -> r = min(2r, 100)
      (u = 4, a sliding window)
      otherwise r unchanged.
    The min/max of the printed equation are read as clamps toward R(1) and
    R(100); the first loss has no predecessor: unchanged.
  * sync accounting (each change of kind synchronises the hot
    rows): one event of hot_bytes per device per swap.
  * the rate persists across epochs.
"""
from __future__ import annotations

import math
from typing import List, Optional, Tuple


def next_rate(r: float, losses: List[float], u: int = 4) -> float:
    """Eq. 5 as read in the module docstring."""
    if len(losses) < 2:
        return r
    if losses[-1] > losses[-2]:
        return max(r / 2.0, 1.0)
    if len(losses) >= u + 1 and all(losses[-k] < losses[-k - 1] for k in range(1, u + 1)):
        return min(r * 2.0, 100.0)
    return r


def phase_len(r: float, n_orig: int) -> int:
    """ceil(r% of a kind's original batch count), at least one batch."""
    return max(1, int(math.ceil(r / 100.0 * n_orig)))


class Scheduler:
    """The scheduler's state machine."""

    def __init__(self, n_cold: int, n_hot: int, r_start: float = 50.0, u: int = 4):
        if not (1.0 <= r_start <= 100.0) or u < 1 or n_cold < 0 or n_hot < 0:
            raise ValueError("bad scheduler arguments")
        self.n = {"cold": n_cold, "hot": n_hot}
        self.r, self.u = float(r_start), u
        self.losses: List[float] = []
        self.rates: List[float] = [self.r]
        self.swaps = 0
        self.sync_events = 0
        self.sync_bytes = 0
        self.new_epoch()

    def new_epoch(self):
        self.done = {"cold": 0, "hot": 0}
        self.next_kind = "cold"           # always begins with cold inputs
        self.last_kind: Optional[str] = None

    def next_phase(self) -> Optional[Tuple[str, int, int]]:
        """(kind, first batch, count), or None once both kinds are drained."""
        k = self.next_kind
        o = "hot" if k == "cold" else "cold"
        if self.done[k] >= self.n[k]:
            k, o = o, k
            if self.done[k] >= self.n[k]:
                return None
        left = self.n[k] - self.done[k]
        cnt = left if self.done[o] >= self.n[o] else min(left, phase_len(self.r, self.n[k]))
        first = self.done[k]
        self.done[k] += cnt
        self.next_kind = o
        self.last_kind = k
        return k, first, cnt

    def pending_swap(self) -> bool:
        """A phase of the other kind follows the one just issued."""
        if self.last_kind is None:
            return False
        o = "hot" if self.last_kind == "cold" else "cold"
        return self.done[o] < self.n[o]

    def record_swap(self, test_loss: float, hot_bytes: int = 0, n_devices: int = 1):
        """Swap boundary: sync accounting, then Eq. 5 with the post-swap loss."""
        self.swaps += 1
        self.sync_events += n_devices
        self.sync_bytes += hot_bytes * n_devices
        self.losses.append(float(test_loss))
        self.r = next_rate(self.r, self.losses, self.u)
        self.rates.append(self.r)


def plan_fixed(n_cold: int, n_hot: int, r: float) -> List[Tuple[str, int]]:
    """The phases at a fixed rate (no loss feedback): [(kind, count), ...]."""
    s = Scheduler(n_cold, n_hot, r)
    out = []
    while True:
        p = s.next_phase()
        if p is None:
            return out
        out.append((p[0], p[2]))
