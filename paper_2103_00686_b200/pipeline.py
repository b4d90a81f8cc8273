"""Orchestration of the FAE hot path over the C ABI (no arithmetic here).

One `FaePipeline` per GPU.  It allocates the device buffers a run needs and
calls, in the paper's order:

  fae_profile   -> per-table loggers k and T             (a1, a2)
  fae_threshold -> hot set + remap                        (a3, a4)
  fae_classify  -> hot/cold ids + remapped hot CSR        (a5, a6)
  fae_extract   -> replicated hot table W_hot             (a7)
  per hot batch: fae_emb_fwd, fae_emb_bwd_update          (a8-a11)

Everything numeric happens inside libfae.so kernels.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import torch

from . import (BUDGET_EXACT, FIXED_T, Ctx, fae_classify, fae_create,
               fae_emb_bwd_update, fae_emb_fwd, fae_extract, fae_group_batches,
               fae_pack_cold, fae_profile, fae_release_scratch, fae_scatter_hot,
               fae_threshold, fae_train_hot_batches)


@dataclasses.dataclass
class Prepared:
    counts: torch.Tensor
    T: List[int]
    n_sampled: int
    thresh: dict
    hot_ids: torch.Tensor
    cold_ids: torch.Tensor
    hot_idx: torch.Tensor
    hot_off: Optional[torch.Tensor]
    packed: dict


class FaePipeline:
    def __init__(self, rows: List[int], dim: int, batch: int, pool: int,
                 max_pool: int = 1, device: int = 0, max_world: int = 1,
                 ctx: Optional[Ctx] = None):
        self.rows = [int(r) for r in rows]
        self.Tn = len(rows)
        self.dim = dim
        self.batch = batch
        self.pool = pool                      # 0 => offsets
        self.device = device
        self.max_pool = max_pool
        max_lookups = batch * self.Tn * max(pool, max_pool, 1)
        self.ctx = ctx or fae_create(device, max_tables=max(self.Tn, 1),
                                     max_rows=sum(self.rows),
                                     max_batch_lookups=max_lookups,
                                     max_batch_bags=batch * self.Tn,
                                     max_dim=max(dim, 4), max_world=max_world)
        self.dev = torch.device("cuda", device)

    # ---------------------------------------------------------------- a1-a7
    def preprocess(self, idx: torch.Tensor, off: Optional[torch.Tensor],
                   n_records: int, x_pct: float = 5.0, seed: int = 1,
                   mode: int = FIXED_T, t: float = 1e-7,
                   budget_bytes: int = 0, small_table_bytes: int = 1 << 20,
                   want_estimate: bool = False,
                   bufs: Optional[Prepared] = None,
                   times: Optional[dict] = None, record_base: int = 0,
                   n_records_global: Optional[int] = None) -> Prepared:
        """times: optional dict accumulating ms per call (the calls return
        host values, so each has synchronised the stream).  record_base /
        n_records_global: this rank's shard of a sharded dataset (global id
        of local record 0, records over all ranks), so the sample is drawn
        from global record ids and equals the unsharded one (fae.h fae_csr)."""
        import time as _t
        dev = self.dev
        t0 = _t.perf_counter()

        def lap(name):
            nonlocal t0
            if times is not None:
                t1 = _t.perf_counter()
                times[name] = times.get(name, 0.0) + (t1 - t0) * 1e3
                t0 = t1
        counts = bufs.counts if bufs else torch.empty(sum(self.rows), dtype=torch.int32, device=dev)
        T, ns = fae_profile(self.ctx, self.rows, self.dim, idx, off, self.pool,
                            n_records, x_pct, seed, counts,
                            record_base=record_base, n_records_global=n_records_global)
        lap("profile")
        th = fae_threshold(self.ctx, self.rows, self.dim, counts, T, x_pct,
                           mode=mode, t=t, budget_bytes=budget_bytes,
                           small_table_bytes=small_table_bytes,
                           want_estimate=want_estimate)
        lap("threshold")
        if bufs is None:
            hot_ids = torch.empty(max(n_records, 1), dtype=torch.int64, device=dev)
            cold_ids = torch.empty(max(n_records, 1), dtype=torch.int64, device=dev)
            hot_idx = torch.empty(max(idx.numel(), 1), dtype=torch.int32, device=dev)
            hot_off = (torch.empty(n_records * self.Tn + 1, dtype=torch.int64, device=dev)
                       if off is not None else None)
        else:
            hot_ids, cold_ids, hot_idx, hot_off = bufs.hot_ids, bufs.cold_ids, bufs.hot_idx, bufs.hot_off
        pk = fae_classify(self.ctx, self.rows, self.dim, idx, off, self.pool,
                          n_records, self.batch, hot_ids, cold_ids, hot_idx, hot_off)
        lap("classify")
        return Prepared(counts, T, ns, th, hot_ids, cold_ids, hot_idx, hot_off, pk)

    def extract(self, W: torch.Tensor, prep: Prepared) -> torch.Tensor:
        """Replicated hot table [H_total, D] (buffer reused across calls)."""
        H = prep.thresh["H_total"]
        buf = getattr(self, "_whot", None)
        if buf is None or buf.shape[0] < max(H, 1):
            buf = torch.empty(max(H, 1), self.dim, dtype=torch.float32, device=self.dev)
            self._whot = buf
        fae_extract(self.ctx, W, buf)
        return buf[:H]

    # ---------------------------------------------------------------- a8-a11
    def batch_args(self, prep: Prepared, i: int):
        """(idx, off, n_bags) views of hot batch i (no copies)."""
        B, Tn = self.batch, self.Tn
        nh = prep.packed["n_hot"]
        r0, r1 = i * B, min((i + 1) * B, nh)
        n_bags = (r1 - r0) * Tn
        if self.pool > 0:
            P = self.pool
            return prep.hot_idx[r0 * Tn * P: r1 * Tn * P], None, n_bags
        return prep.hot_idx, prep.hot_off[r0 * Tn: r1 * Tn + 1], n_bags

    def group(self, prep: Prepared):
        """Sort-and-segment of every hot batch, once (fae_group_batches)."""
        pk = prep.packed
        fae_group_batches(self.ctx, self.rows, self.dim, prep.hot_idx, prep.hot_off,
                          pk["n_hot"], pk["n_hot_lookups"], self.pool, self.batch,
                          prep.thresh["H_total"])

    def train(self, W_hot, first: int, n: int, dY, Y, lr: float):
        """Hot batches [first, first+n) through the graph-replayed loop."""
        fae_train_hot_batches(self.ctx, W_hot, first, n, dY, Y, lr)

    def step(self, W_hot, prep: Prepared, i: int, Y, dY, lr: float):
        idx, off, n_bags = self.batch_args(prep, i)
        fae_emb_fwd(self.ctx, W_hot, idx, off, self.pool, n_bags, Y)
        fae_emb_bwd_update(self.ctx, W_hot, idx, off, self.pool, n_bags, dY, lr)


class MixedEpoch:
    """Hot AND cold mini-batches of one epoch (P:L146,
    L223-230, L299-302, L540).

    Hot batches train the replicated hot table W_hot through the pipeline's
    ctx (grouped once); cold batches train the full master tables W (HBM
    resident: B200 holds the tables the paper keeps in CPU memory) through a
    second ctx that groups the cold CSR in global row ids once (fae_pack_cold
    + fae_group_batches with H = sum N_z), so both kinds run the same
    graph-replayed step.  At every change of kind the hot rows are
    synchronised (the paper's "embedding sync"): hot -> cold writes W_hot
    back into W (fae_scatter_hot), cold -> hot re-extracts W_hot from W
    (fae_extract).  Sequential SGD semantics over the phase order."""

    def __init__(self, pipe: "FaePipeline", prep: Prepared, W: torch.Tensor,
                 idx: torch.Tensor, off: Optional[torch.Tensor], n_records: int,
                 W_hot: torch.Tensor):
        self.pipe, self.prep, self.W, self.W_hot = pipe, prep, W, W_hot
        pk = prep.packed
        self.n_cold = int(pk["n_cold"])
        Tn, B = pipe.Tn, pipe.batch
        n_lookups = int(idx.numel()) if off is None else int(off[-1].item())
        self.n_cold_lookups = n_lookups - int(pk["n_hot_lookups"])
        dev = pipe.dev
        self.cold_idx = torch.empty(max(self.n_cold_lookups, 1), dtype=torch.int32, device=dev)
        self.cold_off = (torch.empty(self.n_cold * Tn + 1, dtype=torch.int64, device=dev)
                         if off is not None else None)
        fae_pack_cold(pipe.ctx, pipe.rows, pipe.dim, idx, pipe.pool, n_records, prep.cold_ids,
                      self.n_cold, self.cold_idx, off=off, cold_off=self.cold_off)
        self.cold = FaePipeline(pipe.rows, pipe.dim, B, pipe.pool,
                                max_pool=getattr(pipe, "max_pool", 1), device=pipe.device)
        self.H_full = sum(pipe.rows)
        if self.n_cold > 0:
            fae_group_batches(self.cold.ctx, pipe.rows, pipe.dim, self.cold_idx, self.cold_off,
                              self.n_cold, self.n_cold_lookups, pipe.pool, B, self.H_full)
            fae_release_scratch(self.cold.ctx)      # two groupings stay alive
        pipe.group(prep)
        fae_release_scratch(pipe.ctx)
        self.n_hot_batches = int(pk["n_hot_batches"])
        self.n_cold_batches = -(-self.n_cold // B)
        self.kind = "hot"          # W_hot holds the current hot rows
        self.swaps = 0

    def swap_to(self, kind: str):
        """Synchronise the hot rows for a phase of `kind` (no-op if current)."""
        if kind == self.kind:
            return
        if kind == "cold":
            fae_scatter_hot(self.pipe.ctx, self.W_hot, self.W)
        else:
            fae_extract(self.pipe.ctx, self.W, self.W_hot)
        self.kind = kind
        self.swaps += 1

    def train(self, kind: str, first: int, n: int, dY, Y, lr: float):
        """Batches [first, first+n) of `kind`, after the swap if needed."""
        self.swap_to(kind)
        if n <= 0:
            return
        if kind == "hot":
            fae_train_hot_batches(self.pipe.ctx, self.W_hot, first, n, dY, Y, lr)
        else:
            fae_train_hot_batches(self.cold.ctx, self.W, first, n, dY, Y, lr)

    def finish(self):
        """Write the hot rows back into W (end of the epoch)."""
        self.swap_to("cold")


class FaeTrainer:
    """FAE training of the DLRM (SURVEY §8(f) NEXT-2 + NEXT-3): the epoch's
    cold and hot mini-batches in the order of the Eq. 5 scheduler
    (P:L538-572), every batch a full DLRM step (a8 -> MLPs / interaction /
    log loss / SGD -> a9 + a10; fae_train_dlrm_batches) — hot batches on the
    replicated hot table, cold batches on the master tables (MixedEpoch) —
    and at every swap boundary the hot rows synchronised and the TEST loss
    of the held-out records evaluated on the master tables and fed to the
    scheduler ("post-swap testing loss").

    dense / label: device [n_records] inputs of the training records (record
    id order); test_idx / test_off / n_test: the held-out records' CSR in
    GLOBAL row ids (fae_pack_cold layout), test_dense / test_label theirs."""

    def __init__(self, ep: MixedEpoch, n_dense: int, bottom, top, params: torch.Tensor,
                 dense: torch.Tensor, label: torch.Tensor, test_idx: torch.Tensor,
                 test_off: Optional[torch.Tensor], n_test: int, test_dense: torch.Tensor,
                 test_label: torch.Tensor, tf32: bool = True):
        from . import Dlrm
        p = ep.pipe
        self.ep, self.params = ep, params
        self.dense, self.label = dense, label
        self.hot_model = Dlrm(p.ctx, n_dense, bottom, top, p.Tn, p.dim, p.batch, tf32=tf32)
        self.cold_model = Dlrm(ep.cold.ctx, n_dense, bottom, top, p.Tn, p.dim, p.batch, tf32=tf32)
        self.test = (test_idx, test_off, int(n_test), test_dense, test_label)
        self.Ybuf = torch.empty(p.batch * p.Tn, p.dim, device=p.dev)

    def train(self, kind: str, first: int, n: int, lr_mlp: float, lr_emb: float):
        ep = self.ep
        ep.swap_to(kind)
        if n <= 0:
            return
        if kind == "hot":
            self.hot_model.train_batches(self.params, ep.W_hot, first, n, ep.prep.hot_ids, self.dense,
                                         self.label, lr_mlp, lr_emb)
        else:
            self.cold_model.train_batches(self.params, ep.W, first, n, ep.prep.cold_ids, self.dense,
                                          self.label, lr_mlp, lr_emb)

    def train_loss(self, reset: bool = True):
        a, n = self.hot_model.loss(reset)
        b, m = self.cold_model.loss(reset)
        return (a + b) / max(n + m, 1.0)

    def test_loss(self) -> float:
        """Mean log loss of the held-out records on the master tables (the
        hot rows written back first)."""
        ep = self.ep
        ep.swap_to("cold")
        idx, off, n_test, tdense, tlabel = self.test
        p = ep.pipe
        B, Tn = p.batch, p.Tn
        model = self.cold_model
        model.loss(reset=True)
        for r0 in range(0, n_test, B):
            r1 = min(r0 + B, n_test)
            nb = (r1 - r0) * Tn
            if off is None:
                bi, bo = idx[r0 * Tn * p.pool: r1 * Tn * p.pool], None
            else:
                bi, bo = idx, off[r0 * Tn: r1 * Tn + 1]
            fae_emb_fwd(ep.cold.ctx, ep.W, bi, bo, p.pool, nb, self.Ybuf[:nb])
            model.step(self.params, r1 - r0, tdense[r0:r1], tlabel[r0:r1], self.Ybuf[:nb], None, 0.0,
                       train=False)
        s, n = model.loss(reset=True)
        return s / max(n, 1.0)

    def run_epoch(self, sched, lr_mlp: float, lr_emb: float, log: Optional[list] = None):
        """One epoch in the scheduler's order; returns the phases run."""
        ep = self.ep
        hot_bytes = ep.prep.thresh["H_total"] * ep.pipe.dim * 4
        phases = []
        while True:
            ph = sched.next_phase()
            if ph is None:
                break
            kind, first, n, swap_after = ph
            self.train(kind, first, n, lr_mlp, lr_emb)
            phases.append((kind, first, n))
            if swap_after:
                tl = self.test_loss()
                sched.record_swap(tl, hot_bytes, 1)
                if log is not None:
                    log.append({"swap": sched.swaps, "after": kind, "batches": n, "test_loss": tl,
                                "rate": sched.rate})
        return phases


__all__ = ["FaePipeline", "Prepared", "MixedEpoch", "FaeTrainer", "FIXED_T", "BUDGET_EXACT"]
