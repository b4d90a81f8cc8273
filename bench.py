"""bench.py — FAE hot path on B200: hot-batch lookups/s (fwd+bwd+update).

One STEP = one pass of the whole hot path over one
batch of synthetic input = this rank's dataset shard:
  fae_profile (sample 5% + loggers) -> fae_threshold (Eq. 1 cutoff, hot set,
  remap) -> fae_classify (hot/cold inputs, packed hot CSR) -> fae_extract
  (replicated hot table) -> every hot mini-batch: fae_emb_fwd +
  fae_emb_bwd_update (+ hot-grad sync over NCCL when N > 1).
value = hot lookups trained by all ranks / max-over-ranks step time.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config terabyte]
       python bench.py --impl reference ...   (CPU oracle arm)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402

METRIC = "hot-batch lookups/sec (fwd+bwd+update) and % of HBM peak at 1/2/4/8 B200"
UNIT = "lookups/s"


NOMINAL_HBM_GBS = 8000.0   # B200 HBM3e nominal (north_star's "~8 TB/s"); frac uses the measured peak


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------
# algorithmic bytes
# ----------------------------------------------------------------------------
def ncu_traffic(kernel, workload):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    of `kernel` from the committed `ncu --set full` summary
    (profiles/ncu_traffic.json, written by tools/ncu_summary.py traffic);
    None when no capture of this kernel on this workload is committed."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        e = t.get(workload, {}).get(kernel)
        return float(e["dram_bytes_per_launch"]) if e else None
    except Exception:
        return None


def fwd_bytes(L, S, D, explicit_off):
    """SURVEY §8(d) algorithmic bytes of a8 per batch: idx 4L [+ offsets
    4(S+1)] + row gathers 4DL + Y write 4DS."""
    return 4 * L + (4 * (S + 1) if explicit_off else 0) + 4 * D * L + 4 * D * S


def bwd_bytes(L, S, U, D, explicit_off):
    """SURVEY §8(d) algorithmic bytes of a9+a10 per batch: idx 4L [+ offsets
    4(S+1)] + dY read once 4DS + one write + read of the 8-byte (key, pos)
    sort pairs 16L + W rows read + write 8DU."""
    return 4 * L + (4 * (S + 1) if explicit_off else 0) + 4 * D * S + 16 * L + 8 * D * U


def design_red_bytes(L, S, U, D):
    """What this design's reduce kernel itself must move (the sort is hoisted
    into the grouping): sorted bag ids 4L, 32-byte segment records 32U, a dY
    row per lookup 4DL, W rows read + write 8DU (reported beside the §8(d)
    figure, never used for frac)."""
    return 4 * L + 32 * U + 4 * D * L + 8 * D * U


def host_info():
    """lscpu-equivalent facts of this host (cpu_baseline's `cores` context)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "usable_cpus": aff}


def pipe_stats(pipe):
    import paper_2103_00686_b200 as fae
    gi = fae.fae_group_info(pipe.ctx)
    return {"segs_per_batch": gi["segments"] / max(gi["n_batches"], 1), **gi}


# ----------------------------------------------------------------------------
# CUDA arm
# ----------------------------------------------------------------------------
def config_of(args):
    import dataclasses
    cfg = gen.CONFIGS[args.config]
    if args.batch:
        cfg = dataclasses.replace(cfg, batch=args.batch)
    return cfg


def run_fae(args):
    import paper_2103_00686_b200 as fae
    from paper_2103_00686_b200.pipeline import FaePipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cfg = config_of(args)
    R = args.records or cfg.records
    Tn, D, B = cfg.n_tables, cfg.dim, cfg.batch
    ds = gen.make_dataset(cfg, n_records=R, device=dev, record_base=rank * R)
    if args.exchange:
        os.environ["FAE_FORCE_MERGE"] = "1"      # read at fae_create
    pipe = FaePipeline(cfg.rows, D, B, cfg.pool, max_pool=max(cfg.pool_hi, 1), device=local,
                       max_world=world)
    # cross-step overlap (one GPU): step k+1's preprocessing and grouping run on
    # a second ctx / stream while step k trains; trainings stay serial (step
    # k+1's extract waits for step k's training on the device)
    overlap = world == 1 and not args.exchange and args.overlap
    pipes, streams = [pipe], [None]
    if overlap:
        pipes.append(FaePipeline(cfg.rows, D, B, cfg.pool, max_pool=max(cfg.pool_hi, 1), device=local,
                                 max_world=world))
        streams = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]
        for p_, s_ in zip(pipes, streams):
            p_.ctx.set_stream(s_)
    if world > 1:
        from paper_2103_00686_b200 import dist as fdist
        fdist.init_comm(pipe.ctx, dev)
    elif args.exchange:                           # the exchange loop on a 1-rank communicator
        fae.fae_comm_init(pipe.ctx, fae.fae_get_nccl_id(), 0, 1)
    W = gen.make_weights(sum(cfg.rows), D, device=dev)
    S_max = B * Tn
    dy_bytes = S_max * D * 4
    n_dy = max(1, math.ceil((args.dy_pool_mb << 20) / dy_bytes))   # > L2: honest dY reads
    dY = gen.make_dy(n_dy * S_max, D, device=dev).view(n_dy, S_max, D)
    Y = torch.empty(S_max, D, device=dev)
    mode = fae.BUDGET_EXACT if cfg.budget_bytes else fae.FIXED_T
    state = {}

    phases = {}

    def mark(name, t0):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        phases[name] = phases.get(name, 0.0) + (t1 - t0) * 1e3
        return t1

    ov = {"train_done": None, "events": []}

    def one_step_ov(k):
        i = k % len(pipes)
        p, st = pipes[i], streams[i]
        with torch.cuda.stream(st):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            e[0].record(st)
            prep = p.preprocess(ds.idx, ds.off, R, x_pct=5.0, seed=args.seed, mode=mode,
                                t=cfg.t, budget_bytes=cfg.budget_bytes,
                                small_table_bytes=cfg.small_bytes, bufs=state.get(("prep", i)),
                                times=phases, record_base=rank * R, n_records_global=world * R)
            state[("prep", i)] = prep
            e[1].record(st)
            p.group(prep)
            e[2].record(st)
            if ov["train_done"] is not None:
                st.wait_event(ov["train_done"])
            W_hot = p.extract(W, prep)
            e[3].record(st)
            p.train(W_hot, 0, prep.packed["n_hot_batches"], dY, Y, args.lr)
            e[4].record(st)
            ov["train_done"] = e[4]
            ov["events"].append(e)
        return prep.packed["n_hot_lookups"], prep

    def one_step():
        if overlap:
            k = state.get("k", 0)
            state["k"] = k + 1
            return one_step_ov(k)
        t = time.perf_counter()
        prep = pipe.preprocess(ds.idx, ds.off, R, x_pct=5.0, seed=args.seed, mode=mode,
                               t=cfg.t, budget_bytes=cfg.budget_bytes,
                               small_table_bytes=cfg.small_bytes, bufs=state.get("prep"),
                               times=phases, record_base=rank * R, n_records_global=world * R)
        state["prep"] = prep
        t = mark("preprocess_total", t)
        pipe.group(prep)
        t = mark("group", t)
        W_hot = pipe.extract(W, prep)
        t = mark("extract", t)
        nb = prep.packed["n_hot_batches"]
        if dist is not None:
            from paper_2103_00686_b200 import dist as fdist
            nb = fdist.max_over_ranks(nb, dev)
        pipe.train(W_hot, 0, nb, dY, Y, args.lr)
        mark("train", t)
        return prep.packed["n_hot_lookups"], prep

    # kernel timing on from the warm-up: the captured training graph (keyed on
    # its buffers, including the timing stamps) is built outside the timed region
    for p_ in pipes:
        fae.fae_set_kernel_timing(p_.ctx, 0 if args.no_ktiming else 1)
    for _ in range(max(args.warmup, len(pipes))):
        one_step()
    torch.cuda.synchronize()
    for p_ in pipes:
        p_.ctx.check()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    l0 = sum(p_.ctx.launches for p_ in pipes)
    phases.clear()
    ov["events"].clear()
    for p_ in pipes:
        fae.fae_set_kernel_timing(p_.ctx, 0 if args.no_ktiming else 1)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    wall0 = time.perf_counter()
    t0.record()
    sev[0].record()
    if overlap:               # the side streams start after t0
        for st_ in streams:
            st_.wait_event(t0)
    hot_lookups = 0
    prep = None
    for k in range(args.steps):
        n, prep = one_step()
        if not overlap:
            sev[k + 1].record()
        hot_lookups += n
    if overlap:               # t1 after both side streams drained
        for st_ in streams:
            torch.cuda.current_stream().wait_stream(st_)
    t1.record()
    torch.cuda.synchronize()
    if overlap:
        ends = [sev[0]] + [e[4] for e in ov["events"]]
        per_step_ms = [ends[k].elapsed_time(ends[k + 1]) for k in range(args.steps)]
        for k, e in enumerate(ov["events"]):
            for name, a, b in (("preprocess_total", 0, 1), ("group", 1, 2), ("extract_and_wait", 2, 3),
                               ("train", 3, 4)):
                phases[name] = phases.get(name, 0.0) + e[a].elapsed_time(e[b])
    else:
        per_step_ms = [sev[k].elapsed_time(sev[k + 1]) for k in range(args.steps)]
    wall = time.perf_counter() - wall0
    ck = clocks.stop()
    for p_ in pipes:
        p_.ctx.check()
    ms = t0.elapsed_time(t1)
    launches = sum(p_.ctx.launches for p_ in pipes) - l0
    kts = [fae.fae_get_kernel_timing(p_.ctx) for p_ in pipes]
    kt = dict(kts[0])
    for k2 in ("fwd", "reduce", "overlap"):
        kt[k2] = (sum(x[k2][0] for x in kts), sum(x[k2][1] for x in kts))
    kt["persist_batches"] = sum(x["persist_batches"] for x in kts)
    xt = fae.fae_get_exchange_timing(pipe.ctx) if (world > 1 or args.exchange) else None
    for p_ in pipes:
        fae.fae_set_kernel_timing(p_.ctx, 0)

    tot = torch.tensor([ms, float(hot_lookups)], dtype=torch.float64, device=dev)
    if dist is not None:
        mx = tot.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tot.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, lookups_all = float(mx[0]), float(sm[1])
    else:
        ms_max, lookups_all = ms, float(hot_lookups)
    peak, kind = peaks()
    res = None
    if rank == 0:
        # dominant kernel of the step, timed live
        fused, persist = kt["fused"], kt["persist"]
        # the dominant kernel of the two-kernel step is the reduce (a9 + a10,
        # the step's HBM traffic: 34 MB of DRAM per Terabyte-shaped launch vs
        # 6 MB for the forward; 62-63 % of the serialised ncu launch list).  Its
        # exclusive share understates it: since the forward runs at 2 CTAs per
        # SM, the reduce's static loads and long-segment sums execute during
        # the forward, whose exclusive share then absorbs them (the forward's
        # own figures are reported beside, `roofline.fwd`)
        kname = "reduce"
        overlap = {"steps_overlapped": kt["overlap"][1],
                   "avg_reduce_entry_lead_us": kt["overlap"][0] / max(kt["overlap"][1], 1) * 1e3}
        kms, kn = kt[kname]
        avg_s = (kms / max(kn, 1)) / 1e3
        L_b = prep.packed["n_hot_lookups"] / max(prep.packed["n_hot_batches"], 1)
        S_b = prep.packed["n_hot"] * Tn / max(prep.packed["n_hot_batches"], 1)
        gi = pipe_stats(pipe)
        U_b = gi["segs_per_batch"]
        F_b = gi["free_segments"] / max(gi["n_batches"], 1)
        expl = cfg.pool == 0
        if fused or persist:   # backward+SGD of one batch + forward of the next
            kb = bwd_bytes(L_b, S_b, U_b, D, expl) + fwd_bytes(L_b, S_b, D, expl)
            kdesign = design_red_bytes(L_b, S_b, U_b, D) + 4 * L_b + 4 * D * S_b + (16 + 4 * D) * F_b
            if persist:        # one launch trains every batch of the call
                kb *= kt["persist_batches"] / max(kn, 1)
                kdesign *= kt["persist_batches"] / max(kn, 1)
        elif kname == "fwd":
            kb = kdesign = fwd_bytes(L_b, S_b, D, expl)
        else:
            kb = bwd_bytes(L_b, S_b, U_b, D, expl)
            kdesign = design_red_bytes(L_b, S_b, U_b, D)
        achieved = kb / avg_s / 1e9 if avg_s > 0 else 0.0
        kname_full = ("k_train_persist" if persist else "k_grp_fused_pdl" if fused else
                      {"fwd": "k_grp_fwd_pdl", "reduce": "k_grp_reduce_pdl"}[kname])
        res = {
            "metric": METRIC, "value": lookups_all / (ms_max / 1e3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "ms_per_step_median": statistics.median(per_step_ms), "per_step_ms": per_step_ms,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Zipf s=1.1, Feistel-scattered rows; gen/)",
            "config": {"workload": f"{cfg.name}-shaped", "records_per_gpu": R,
                       "tables": Tn, "rows_total": sum(cfg.rows), "dim": D,
                       "batch_per_gpu": B, "pooling": cfg.pool or f"U{{{cfg.pool_lo}..{cfg.pool_hi}}}",
                       "threshold": ({"budget_bytes": cfg.budget_bytes} if cfg.budget_bytes else {"t": cfg.t}),
                       "x_pct": 5.0, "lr": args.lr,
                       "hot_rows": prep.thresh["H_total"], "hot_records": prep.packed["n_hot"],
                       "hot_batches_per_step": prep.packed["n_hot_batches"],
                       "hot_lookups_per_step": prep.packed["n_hot_lookups"],
                       "distinct_rows_per_batch": U_b,
                       "l2": "inputs > L2 (dataset %.1f GB, dY pool %d MB)" % (
                           ds.idx.numel() * 4 / 1e9, n_dy * dy_bytes >> 20),
                       "parallelism": f"dp{world}",
                       "cross_step_overlap": (("step k+1's preprocessing + grouping on a second ctx / stream "
                                               "while step k trains; trainings serial") if overlap else None)},
            "gpu_launches": launches,
            "roofline": {"kernel": kname_full,
                         "timing": ("CUDA events around each cooperative launch on the ctx stream, every launch "
                                    "of the timed region" if persist else
                                    "in-kernel globaltimer, exclusive share of the step, every launch of the timed region"),
                         "bound": "hbm", "achieved": achieved,
                         "peak": peak, "peak_kind": kind, "unit": "GB/s",
                         "frac": achieved / peak,
                         # report the nominal-basis fraction too (north_star's ~8 TB/s)
                         "frac_nominal": achieved / NOMINAL_HBM_GBS, "peak_nominal": NOMINAL_HBM_GBS,
                         "traffic": ncu_traffic(kname_full, f"{cfg.name}-shaped"),
                         "bytes_per_launch": kb,
                         "bytes_formula": ("SURVEY §8(d): fwd 4L+4DL+4DS [+4(S+1)], bwd+update "
                                           "4L+4DS+16L+8DU [+4(S+1)]; per-batch L, S, U measured"),
                         "per_batch": {"L": L_b, "S": S_b, "U": U_b, "F": F_b},
                         "design_bytes_per_launch": kdesign,
                         "design_frac": (kdesign / avg_s / 1e9) / peak if avg_s > 0 else 0.0,
                         "avg_launch_us": avg_s * 1e6,
                         "kernels_us": {k: (kt[k][0] / max(kt[k][1], 1)) * 1e3 for k in ("fwd", "reduce")},
                         "launches_timed": kn,
                         **({} if (fused or persist) else {"fwd": (lambda fb, fu: {
                             "kernel": "k_grp_fwd_pdl", "bytes_per_launch": fb, "avg_launch_us": fu,
                             "achieved": fb / (fu * 1e-6) / 1e9 if fu else None,
                             "frac": (fb / (fu * 1e-6) / 1e9) / peak if fu else None,
                             "traffic": ncu_traffic("k_grp_fwd_pdl", f"{cfg.name}-shaped"),
                             "note": "exclusive share includes the reduce's pre-wait work that overlaps it; "
                                     "the Zipf head of W_hot is served by L2"})(
                             fwd_bytes(L_b, S_b, D, expl), (kt["fwd"][0] / max(kt["fwd"][1], 1)) * 1e3)}),
                         # the whole a8-a10 step per batch (fwd + bwd + update) on §8(d) bytes
                         # over the training loop's time per batch (every kernel of the step)
                         "step": (lambda sb, su: {"bytes_per_batch": sb, "us_per_batch": su,
                                                  "achieved": sb / (su * 1e-6) / 1e9 if su else None,
                                                  "frac": (sb / (su * 1e-6) / 1e9) / peak if su else None})(
                             fwd_bytes(L_b, S_b, D, expl) + bwd_bytes(L_b, S_b, U_b, D, expl),
                             phases.get("train", 0.0) / args.steps * 1e3 / max(prep.packed["n_hot_batches"], 1)),
                         **({"batches_per_launch": kt["persist_batches"] / max(kn, 1),
                             "us_per_batch": avg_s * 1e6 * kn / max(kt["persist_batches"], 1)}
                            if persist else {"pdl": overlap})},
            "clocks": ck,
            "wall_s": wall,
            "phases_ms_per_step": {k: v / args.steps for k, v in phases.items()},
            **({"sync": sync_report(xt, world, D, kt)} if xt else {}),
            # the a8-a10 training loop alone (the value above times the whole
            # hot path a1-a10 per step)
            "train_only_lookups_per_s": (lookups_all / (phases["train"] / 1e3)
                                         if phases.get("train") else None),
        }
    return res, (pipe, ds, W, cfg, R, dist, rank, world, dev, dY, Y, pipes, streams)


def sync_report(xt, world, D, kt):
    """a11 exchange per training step, device-timed on rank 0:
    every rank contributes xcap (row, G) entries of 4 + 4D bytes (xcap = the
    largest U of any rank and step) and receives world-1 of them; nccl-tests
    conventions: allgather algBW = world * slot bytes / time, busBW = algBW *
    (world-1)/world, against NVLink 5's 900 GB/s per direction."""
    st = max(xt["steps_timed"], 1)
    slot = xt["slot_bytes"] / max(xt["steps"], 1)
    ag_s = xt["allgather_ms"] / st / 1e3
    algbw = world * slot / ag_s / 1e9 if ag_s > 0 else None
    busbw = algbw * (world - 1) / world if algbw else None
    step_us = ((kt["fwd"][0] + kt["reduce"][0]) / max(kt["reduce"][1], 1)) * 1e3 + \
        (xt["allgather_ms"] + xt["merge_ms"]) / st * 1e3
    return {"transport": "nccl", "xcap_entries": xt["xcap"],
            "slot_bytes_per_step": slot, "recv_bytes_per_gpu_per_step": (world - 1) * slot,
            "allgather_us_per_step": ag_s * 1e6, "merge_us_per_step": xt["merge_ms"] / st * 1e3,
            "train_step_us": step_us,
            "algbw_GBs": algbw, "busbw_GBs": busbw,
            "busbw_frac_of_900": (busbw / 900.0) if busbw else None,
            "timing": "in-kernel globaltimer: reduce-emit end -> first merge CTA (all-gather), merge CTAs"}


def run_e2e(args, ctxs):
    """Same metric through the public API with HOST inputs: every step copies
    its dataset shard (the step's input records) from pinned host memory,
    double-buffered on a copy stream so step k+1's copy overlaps step k's
    compute once step k has classified its records; the embedding tables are
    model state and stay resident in HBM between steps (as in the device
    run); the trained hot table (the step's result) is read back into pinned
    host memory every step."""
    import paper_2103_00686_b200 as fae
    pipe, ds, W, cfg, R, dist, rank, world, dev, dY, Y, pipes, streams = ctxs
    idx_h = ds.idx.cpu().pin_memory()
    off_h = ds.off.cpu().pin_memory() if ds.off is not None else None
    del ds
    idx_d = [torch.empty(idx_h.shape, dtype=idx_h.dtype, device=dev) for _ in range(2)]
    off_d = [torch.empty(off_h.shape, dtype=off_h.dtype, device=dev) for _ in range(2)] if off_h is not None else None
    copy_s = torch.cuda.Stream(device=dev)
    rb_s = torch.cuda.Stream(device=dev)
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    for e in free:
        e.record()
    mode = fae.BUDGET_EXACT if cfg.budget_bytes else fae.FIXED_T
    st = {}
    npipe = len(pipes)

    CH = 16 << 20   # elements per chunk (64 MB): the small host<->device copies of
    #                  the compute path interleave with the big input copy

    def enqueue_copy(k):
        b = k % 2
        with torch.cuda.stream(copy_s):
            copy_s.wait_event(free[b])
            for src, dst in ([(idx_h, idx_d[b])] + ([(off_h, off_d[b])] if off_h is not None else [])):
                for c0 in range(0, src.numel(), CH):
                    dst[c0:c0 + CH].copy_(src[c0:c0 + CH], non_blocking=True)
            ready[b].record(copy_s)

    trace = os.environ.get("FAE_E2E_TRACE") is not None

    def mark(tag, t_prev, s_):
        if not trace:
            return t_prev
        s_.synchronize()
        t = time.perf_counter()
        print(f"[e2e] {tag:10s} {(t - t_prev) * 1e3:8.2f} ms", file=sys.stderr)
        return t

    def step(k, last):
        b = k % 2
        i = k % npipe
        p = pipes[i]
        s_ = streams[i] if streams[i] is not None else torch.cuda.current_stream()
        tt = time.perf_counter()
        with torch.cuda.stream(s_):
            s_.wait_event(ready[b])
            tt = mark("wait-in", tt, s_)
            prep = p.preprocess(idx_d[b], off_d[b] if off_d is not None else None, R, x_pct=5.0,
                                seed=args.seed, mode=mode, t=cfg.t, budget_bytes=cfg.budget_bytes,
                                small_table_bytes=cfg.small_bytes, bufs=st.get(("prep", i)),
                                record_base=rank * R, n_records_global=world * R)
            tt = mark("preprocess", tt, s_)
            free[b].record(s_)          # the hot CSR is built: this input buffer is free
            st[("prep", i)] = prep
            p.group(prep)
            tt = mark("group", tt, s_)
            if not last:
                # next step's input crosses PCIe during this step's extract + train
                # (after the grouping, whose small host copies would queue behind it)
                enqueue_copy(k + 1)
            if ("rb_done", i) in st:    # this pipe's previous readback still reads its hot table
                s_.wait_event(st[("rb_done", i)])
            if "train_done" in st:      # trainings stay in sequence
                s_.wait_event(st["train_done"])
            W_hot = p.extract(W, prep)
            nb = prep.packed["n_hot_batches"]
            if dist is not None:
                from paper_2103_00686_b200 import dist as fdist
                nb = fdist.max_over_ranks(nb, dev)
            p.train(W_hot, 0, nb, dY, Y, args.lr)
            trained = torch.cuda.Event()
            trained.record(s_)
            st["train_done"] = trained
            tt = mark("train", tt, s_)
        if ("out", i) not in st or st[("out", i)].numel() < W_hot.numel():
            st[("out", i)] = torch.empty(W_hot.numel() + W_hot.numel() // 4, dtype=W_hot.dtype).pin_memory()
        out = st[("out", i)][:W_hot.numel()].view_as(W_hot)
        # the trained hot table back to host memory on its own stream, so it
        # overlaps the next steps (this pipe's next extract waits for it)
        with torch.cuda.stream(rb_s):
            rb_s.wait_event(trained)
            out.copy_(W_hot, non_blocking=True)
            st[("rb_done", i)] = torch.cuda.Event()
            st[("rb_done", i)].record(rb_s)
        mark("readback", tt, rb_s)
        h2d = idx_h.numel() * 4 + (off_h.numel() * 8 if off_h is not None else 0)
        return prep.packed["n_hot_lookups"], h2d, out.numel() * 4

    enqueue_copy(0)
    step(0, True)             # warm-up
    torch.cuda.synchronize()
    ksteps = max(5, args.steps)   # amortise the first (unoverlapped) input copy
    t0 = time.perf_counter()
    n = h2d = d2h = 0
    enqueue_copy(0)
    for k in range(ksteps):
        a, b, c = step(k, k == ksteps - 1)
        n += a
        h2d, d2h = b, c
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tot = torch.tensor([dt, float(n)], dtype=torch.float64, device=dev)
    if dist is not None:
        mx = tot.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tot.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        dt, n = float(mx[0]), float(sm[1])
    return {"value": n / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": ksteps,
            "overlap": ("step k+1's input copy runs on a copy stream during step k's extract/train; the hot-table "
                        "readback runs on its own stream during step k+1's preprocessing")}


# ----------------------------------------------------------------------------
# CPU oracle arm (cpu_baseline and --impl reference)
# ----------------------------------------------------------------------------
def oracle_step(cfg, R_s, max_batches, seed, lr, ds):
    """The oracle, as it stands, over a bounded sample of the workload:
    the full a1-a10 pipeline on the first R_s records (sample, loggers,
    threshold, remap, classify, pack, then at most max_batches hot batches of
    fwd + bwd + SGD).  The hot table's rows are drawn by counter
    (gen.make_weight_rows: the same bits as extracting them from the full
    table, which at Terabyte shape is 48 GB).  Returns (hot lookups trained,
    seconds)."""
    import numpy as np
    import oracle
    t0 = time.perf_counter()
    x = 5.0
    samp = oracle.sample(R_s, x, seed)
    counts, T, _ = oracle.histogram(ds.rows, ds.idx, ds.off, ds.fixed_pool, R_s, samp)
    small = cfg.small_bytes
    if cfg.budget_bytes:
        r = oracle.budget_exact(ds.rows, cfg.dim, small, counts, T, x, cfg.budget_bytes)
        kmin = r["kmin"]
    else:
        kmin = oracle.kmin_fixed_t(ds.rows, cfg.dim, small, T, cfg.t, x)
    hot = oracle.tag_rows(ds.rows, cfg.dim, small, counts, kmin)
    rm, base, H = oracle.remap(ds.rows, hot)
    flag = oracle.classify(ds.rows, ds.idx, ds.off, ds.fixed_pool, R_s, rm)
    pk = oracle.pack(ds.rows, ds.idx, ds.off, ds.fixed_pool, R_s, rm, flag)
    B, Tn = cfg.batch, cfg.n_tables
    nb = min(max_batches, -(-pk["n_hot"] // B))
    t_gen = time.perf_counter()                  # input generation: not timed
    W_hot = gen.make_weight_rows(torch.from_numpy(np.nonzero(rm >= 0)[0]), cfg.dim).numpy()
    dys = [gen.make_dy(B * Tn, cfg.dim, seed=1000 + i).numpy() for i in range(max(1, min(nb, 8)))]
    t_gen = time.perf_counter() - t_gen
    slot = np.full(max(H, 1), -1, np.int32)
    done = 0
    for i in range(nb):
        r0, r1 = i * B, min((i + 1) * B, pk["n_hot"])
        n_bags = (r1 - r0) * Tn
        if ds.off is None:
            P = ds.fixed_pool
            bi = pk["hot_idx"][r0 * Tn * P: r1 * Tn * P]
            off = None
        else:
            P = 0
            off = pk["hot_off"][r0 * Tn: r1 * Tn + 1]
            bi = pk["hot_idx"]
        dY = dys[i % len(dys)][:n_bags]
        oracle.emb_fwd(W_hot, bi, off, P, n_bags)
        W_hot, _ = oracle.emb_bwd_sgd(W_hot, bi, off, P, n_bags, dY, lr, slot)
        done += (r1 - r0) * Tn * P if off is None else int(off[-1] - off[0])
    return done, time.perf_counter() - t0 - t_gen


CPU_DEFAULTS = {   # records / hot batches of the bounded oracle sample (~10-30 s)
    "tiny": (10_000, 1000), "kaggle": (4_000_000, 400), "terabyte": (3_000_000, 120),
    "alibaba": (1_000_000, 200)}


def oracle_sample_setup(cfg, R_s):
    """The first R_s records of the workload (drawn on the GPU when there is
    one — the generators give the same bits on either device)."""
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    ds = gen.make_dataset(cfg, n_records=R_s, device=dev)
    return ds.to("cpu")


def cpu_runs(cfg, args, variants=("serial", "omp")):
    import oracle
    R_s = min(args.cpu_records or CPU_DEFAULTS[cfg.name][0], cfg.records)
    nbat = args.cpu_batches or CPU_DEFAULTS[cfg.name][1]
    ds = oracle_sample_setup(cfg, R_s)
    out = {}
    for v in variants:
        oracle.use_omp(v == "omp")
        try:
            n, dt = oracle_step(cfg, R_s, nbat, args.seed, args.lr, ds)
        finally:
            oracle.use_omp(False)
        out[v] = (n, dt, oracle.omp_threads() if v == "omp" else 1)
    return R_s, nbat, out


def cpu_baseline(cfg, args):
    R_s, nbat, runs = cpu_runs(cfg, args)
    n, dt, cores = runs["omp"]
    n1, dt1, _ = runs["serial"]
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"full a1-a10 oracle pipeline (fp64 C, OpenMP build, {cores} threads) on the first "
                      f"{R_s} records of the {cfg.name}-shaped workload, <= {nbat} hot batches trained "
                      f"({n} hot lookups in {dt:.1f} s)",
            "single_thread": {"value": n1 / dt1, "cores": 1, "seconds": dt1},
            "host": host_info()}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle
    cfg = gen.CONFIGS[args.config]
    # each step a bounded sample so that the whole --steps K --warmup W run
    # ends within a few minutes
    R_s = min(args.ref_records, cfg.records)
    ds = oracle_sample_setup(cfg, R_s)
    oracle.use_omp(True)
    try:
        for _ in range(args.warmup):
            oracle_step(cfg, R_s, args.ref_batches, args.seed, args.lr, ds)
        n_tot, t_tot = 0, 0.0
        for _ in range(args.steps):
            n, dt = oracle_step(cfg, R_s, args.ref_batches, args.seed, args.lr, ds)
            n_tot += n
            t_tot += dt
    finally:
        oracle.use_omp(False)
    cores = oracle.omp_threads()
    v = n_tot / t_tot
    samp = (f"full a1-a10 oracle pipeline on the first {R_s} records, <= {args.ref_batches} "
            f"hot batches per step, fp64 C (OpenMP build, {cores} threads)")
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_tot * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Zipf s=1.1; gen/)",
            "config": {"workload": f"{cfg.name}-shaped", "records_per_step": R_s},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": samp,
                             "host": host_info()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_sweep(args):
    """Threshold sweep (BASELINE.json configs[4]; P:L331-342
    fig:hotinputembsize): BUDGET_EXACT with L = f * sum N_z * D * 4
    for hot-row fractions f, on one GPU.  Per point: the hot set actually
    chosen (the 5% sample bounds it: a row never sampled is never hot, R25),
    the hot-input share, the per-batch distinct rows U, the training loop's
    lookups/s, and the a11 exchange each GPU would receive per step at
    G = 2 / 4 / 8 (padded all-gather: (G-1) * U * (4 + 4D) bytes) with its
    NVLink lower bound at 900 GB/s.  Prints one JSON line."""
    import paper_2103_00686_b200 as fae
    from paper_2103_00686_b200.pipeline import FaePipeline
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    out = []
    for name in args.sweep_configs.split(","):
        cfg = gen.CONFIGS[name]
        R = args.records or cfg.records
        Tn, D, B = cfg.n_tables, cfg.dim, cfg.batch
        ds = gen.make_dataset(cfg, n_records=R, device=dev)
        W = gen.make_weights(sum(cfg.rows), D, device=dev)
        S = B * Tn
        n_dy = max(1, math.ceil((args.dy_pool_mb << 20) / (S * D * 4)))
        dY = gen.make_dy(n_dy * S, D, device=dev).view(n_dy, S, D)
        Y = torch.empty(S, D, device=dev)
        pipe = FaePipeline(cfg.rows, D, B, cfg.pool, max_pool=max(cfg.pool_hi, 1), device=0)
        rows_total = sum(cfg.rows)
        for f in [float(v) for v in args.sweep_fracs.split(",")]:
            budget = int(f / 100.0 * rows_total * D * 4)
            t0 = time.perf_counter()
            prep = pipe.preprocess(ds.idx, ds.off, R, x_pct=5.0, seed=args.seed, mode=fae.BUDGET_EXACT,
                                   budget_bytes=budget, small_table_bytes=cfg.small_bytes)
            pipe.group(prep)
            W_hot = pipe.extract(W, prep)
            torch.cuda.synchronize()
            pre_ms = (time.perf_counter() - t0) * 1e3
            nb = prep.packed["n_hot_batches"]
            pipe.train(W_hot, 0, nb, dY, Y, args.lr)            # warm-up (graph capture)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pipe.train(W_hot, 0, nb, dY, Y, args.lr)
            e1.record()
            torch.cuda.synchronize()
            pipe.ctx.check()
            tr_ms = e0.elapsed_time(e1)
            gi = fae.fae_group_info(pipe.ctx)
            U = gi["segments"] / max(gi["n_batches"], 1)
            H = prep.thresh["H_total"]
            sync = {str(G): {"bytes_per_gpu_per_step": (G - 1) * U * (4 + 4 * D),
                             "nvlink_floor_us": (G - 1) * U * (4 + 4 * D) / 900e9 * 1e6} for G in (2, 4, 8)}
            out.append({"workload": f"{name}-shaped", "f_pct": f, "budget_bytes": budget,
                        "hot_rows": H, "hot_rows_pct": 100.0 * H / rows_total,
                        "budget_slack": prep.thresh["budget_slack"], "K": prep.thresh["K"],
                        "hot_records_pct": 100.0 * prep.packed["n_hot"] / R,
                        "hot_lookups_pct": 100.0 * prep.packed["n_hot_lookups"] / max(ds.n_lookups, 1),
                        "hot_batches": nb, "U_per_batch": U,
                        "preprocess_ms": pre_ms, "train_ms": tr_ms,
                        "train_lookups_per_s": prep.packed["n_hot_lookups"] / (tr_ms / 1e3) if tr_ms else None,
                        "us_per_batch": tr_ms * 1e3 / max(nb, 1), "sync": sync})
            print(json.dumps(out[-1]), file=sys.stderr, flush=True)
        del ds, W, dY, pipe
        torch.cuda.empty_cache()
    print(json.dumps({"sweep": out, "records_per_gpu": {n: args.records or gen.CONFIGS[n].records
                                                        for n in args.sweep_configs.split(",")}}), flush=True)


def run_mixed(args):
    """NEXT-1 timed mixed epoch (P:L146, L223-230, L299-302,
    L540): every hot AND cold mini-batch of one GPU's dataset, cold first,
    in phases of ceil(r% of each kind's batch count) (the paper's R(r),
    P:L553-572; fixed rate here), the hot rows synchronised at every change
    of kind.  Cold batches train the HBM-resident master tables through the
    same grouped, graph-replayed step (pipeline.MixedEpoch).  Device-timed
    phases and swaps (CUDA events); one JSON line, not the driver's bench."""
    import paper_2103_00686_b200 as fae
    from paper_2103_00686_b200.pipeline import FaePipeline, MixedEpoch
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    cfg = config_of(args)
    R = args.records or cfg.records
    Tn, D, B = cfg.n_tables, cfg.dim, cfg.batch
    ds = gen.make_dataset(cfg, n_records=R, device=dev)
    W = gen.make_weights(sum(cfg.rows), D, device=dev)
    S = B * Tn
    n_dy = max(1, math.ceil((args.dy_pool_mb << 20) / (S * D * 4)))
    dY = gen.make_dy(n_dy * S, D, device=dev).view(n_dy, S, D)
    Y = torch.empty(S, D, device=dev)
    pipe = FaePipeline(cfg.rows, D, B, cfg.pool, max_pool=max(cfg.pool_hi, 1), device=0)
    mode = fae.BUDGET_EXACT if cfg.budget_bytes else fae.FIXED_T
    prep = pipe.preprocess(ds.idx, ds.off, R, x_pct=5.0, seed=args.seed, mode=mode, t=cfg.t,
                           budget_bytes=cfg.budget_bytes, small_table_bytes=cfg.small_bytes)
    W_hot = pipe.extract(W, prep)
    t0 = time.perf_counter()
    ep = MixedEpoch(pipe, prep, W, ds.idx, ds.off, R, W_hot)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t0) * 1e3
    nh, nc = ep.n_hot_batches, ep.n_cold_batches
    r = args.rate
    ph, pc = max(1, math.ceil(nh * r / 100)), max(1, math.ceil(nc * r / 100))
    plan, fh, fc = [], 0, 0
    while fh < nh or fc < nc:             # cold first, alternate until both drain
        if fc < nc:
            plan.append(("cold", fc, min(pc, nc - fc)))
            fc += plan[-1][2]
        if fh < nh:
            plan.append(("hot", fh, min(ph, nh - fh)))
            fh += plan[-1][2]
    ep.train("hot", 0, 0, dY, Y, args.lr)
    for kind, first, n in plan[:4]:       # warm-up: graph capture of both loops
        ep.train(kind, first, min(n, 2 * 128), dY, Y, args.lr)
    ep.swap_to("hot")
    torch.cuda.synchronize()
    ev = []
    res = {"hot_ms": 0.0, "cold_ms": 0.0, "swap_to_cold_ms": 0.0, "swap_to_hot_ms": 0.0}
    sw0 = ep.swaps
    start = torch.cuda.Event(enable_timing=True)
    start.record()
    prev = start
    for kind, first, n in plan:
        a = torch.cuda.Event(enable_timing=True)
        ep.swap_to(kind)
        a.record()
        b = torch.cuda.Event(enable_timing=True)
        ep.train(kind, first, n, dY, Y, args.lr)
        b.record()
        ev.append((kind, prev, a, b))
        prev = b
    a = torch.cuda.Event(enable_timing=True)
    ep.finish()
    a.record()
    torch.cuda.synchronize()
    pipe.ctx.check()
    ep.cold.ctx.check()
    for kind, p0, a0, b0 in ev:          # every phase begins with a change of kind
        res["swap_to_" + kind + "_ms"] += p0.elapsed_time(a0)
        res[kind + "_ms"] += a0.elapsed_time(b0)
    res["swap_to_cold_ms"] += prev.elapsed_time(a)
    total = start.elapsed_time(a)
    hl, cl = prep.packed["n_hot_lookups"], ep.n_cold_lookups
    swaps = ep.swaps - sw0
    hot_bytes = prep.thresh["H_total"] * D * 4
    out = {"mode": "mixed-epoch", "workload": f"{cfg.name}-shaped", "records": R, "rate_pct": r,
           "phases": len(plan), "swaps": swaps, "hot_batches": nh, "cold_batches": nc,
           "hot_lookups": hl, "cold_lookups": cl, "hot_rows": prep.thresh["H_total"],
           "hot_table_bytes": hot_bytes, "epoch_ms": total,
           "epoch_lookups_per_s": (hl + cl) / (total / 1e3),
           "hot_us_per_batch": res["hot_ms"] * 1e3 / max(nh, 1),
           "cold_us_per_batch": res["cold_ms"] * 1e3 / max(nc, 1),
           "swap_ms_total": res["swap_to_cold_ms"] + res["swap_to_hot_ms"],
           "swap_share": (res["swap_to_cold_ms"] + res["swap_to_hot_ms"]) / total,
           "swap_ms_each": (res["swap_to_cold_ms"] + res["swap_to_hot_ms"]) / max(swaps, 1),
           "sync_bytes_per_swap": hot_bytes, **res, "setup_ms": setup_ms,
           "timing": "CUDA events on the ctx stream around each swap and phase"}
    print(json.dumps(out), flush=True)


# tab:benchmarks: RMC2 (Kaggle) / RMC3 (Terabyte) DLRM widths
DLRM_MODELS = {"kaggle": (13, [512, 256, 64, 16], [512, 256, 1]),
               "terabyte": (13, [512, 256, 64], [512, 512, 256, 1])}


def run_train(args):
    """NEXT-2 + NEXT-3: one epoch of FAE training of the paper's DLRM
    (RMC2 Kaggle / RMC3 Terabyte widths, tab:benchmarks) on one GPU: every
    cold and hot mini-batch of the dataset in the Eq. 5 scheduler's order
    (cold first, R(--rate) start), each a full DLRM step (a8, MLPs on TF32
    tensor cores, interaction, log loss, SGD, a9 + a10), hot rows
    synchronised and the test loss of held-out records evaluated at every
    swap.  Device-timed (CUDA events); one JSON line, not the driver's bench."""
    import paper_2103_00686_b200 as fae
    from paper_2103_00686_b200.pipeline import FaePipeline, FaeTrainer, MixedEpoch
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    cfg = config_of(args)
    if cfg.name not in DLRM_MODELS:
        raise SystemExit(f"--train: no DLRM model for {cfg.name} (RMC1 is TBSM, out of scope)")
    n_dense, bottom, top = DLRM_MODELS[cfg.name]
    R = args.records or cfg.records
    Tn, D, B = cfg.n_tables, cfg.dim, cfg.batch
    ds = gen.make_dataset(cfg, n_records=R, device=dev)
    W = gen.make_weights(sum(cfg.rows), D, device=dev)
    pipe = FaePipeline(cfg.rows, D, B, cfg.pool, max_pool=max(cfg.pool_hi, 1), device=0)
    mode = fae.BUDGET_EXACT if cfg.budget_bytes else fae.FIXED_T
    t0 = time.perf_counter()
    prep = pipe.preprocess(ds.idx, ds.off, R, x_pct=5.0, seed=args.seed, mode=mode, t=cfg.t,
                           budget_bytes=cfg.budget_bytes, small_table_bytes=cfg.small_bytes)
    W_hot = pipe.extract(W, prep)
    ep = MixedEpoch(pipe, prep, W, ds.idx, ds.off, R, W_hot)
    torch.cuda.synchronize()
    prep_ms = (time.perf_counter() - t0) * 1e3
    dims = gen.dlrm_dims(n_dense, bottom, top, Tn, D)
    params = gen.dlrm_pad(gen.make_dlrm_params(dims, device=dev), dims)
    dense = gen.make_dense(R, n_dense, device=dev)
    label = gen.make_labels(R, n_dense, device=dev)
    n_test = args.test_records
    tds = gen.make_dataset(cfg, n_records=n_test, device=dev, record_base=R)
    gbase = torch.tensor([0] + list(__import__("itertools").accumulate(cfg.rows))[:-1], device=dev)
    tidx = (tds.idx.view(n_test, Tn) + gbase).view(-1).to(torch.int32)
    tr = FaeTrainer(ep, n_dense, bottom, top, params, dense, label, tidx, None, n_test,
                    gen.make_dense(n_test, n_dense, device=dev, record_base=R),
                    gen.make_labels(n_test, n_dense, device=dev, record_base=R), tf32=True)
    nh, nc = ep.n_hot_batches, ep.n_cold_batches
    # warm-up: capture both loops' graphs and run a few batches (then restore)
    p_save, W_save, Wh_save = params.clone(), W.clone(), W_hot.clone()
    tr.train("cold", 0, min(nc, 256), args.lr_mlp, args.lr)
    tr.train("hot", 0, min(nh, 256), args.lr_mlp, args.lr)
    tr.test_loss()
    ep.swap_to("hot")
    params.copy_(p_save)
    W.copy_(W_save)
    W_hot.copy_(Wh_save)
    del p_save, W_save, Wh_save
    tr.train_loss(reset=True)
    loss0 = tr.test_loss()
    ep.swap_to("hot")
    sched = fae.Scheduler(nc, nh, args.rate)
    log = []
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    phases = tr.run_epoch(sched, args.lr_mlp, args.lr, log)
    ep.finish()
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    pipe.ctx.check()
    ep.cold.ctx.check()
    ms = e0.elapsed_time(e1)
    train_loss = tr.train_loss(reset=True)
    loss1 = tr.test_loss()
    hl, cl = prep.packed["n_hot_lookups"], ep.n_cold_lookups
    fl = 6 * sum(i * o for i, o in dims) * R      # fwd 2, bwd 4 flops per weight per sample
    peak_bf16 = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        peak_bf16 = float(pk.get("bf16_tflops") or pk.get("bf16_dense_tflops") or 0) or None
    except Exception:
        pass
    out = {"mode": "fae-train-epoch", "workload": f"{cfg.name}-shaped", "model": {
               "n_dense": n_dense, "bottom": bottom, "top": top, "interaction": "dot",
               "params": int(params.numel()), "gemm": "cuBLAS TF32 tensor cores, fp32 master weights"},
           "records": R, "hot_records": prep.packed["n_hot"], "hot_batches": nh, "cold_batches": nc,
           "batch": B, "rate_start": args.rate, "phases": len(phases), "swaps": sched.swaps,
           "sync_bytes": int(sched.s.sync_bytes), "epoch_ms": ms, "wall_s": wall,
           "samples_per_s": R / (ms / 1e3), "lookups_per_s": (hl + cl) / (ms / 1e3),
           "us_per_batch": ms * 1e3 / (nh + nc), "mlp_tflops": fl / (ms / 1e3) / 1e12,
           "mlp_peak_tf32_tflops": (peak_bf16 / 2 if peak_bf16 else None),
           "test_loss_before": loss0, "test_loss_after": loss1, "train_loss_epoch": train_loss,
           "swap_log": log[:64], "preprocess_ms": prep_ms, "n_test": n_test,
           "lr_mlp": args.lr_mlp, "lr_emb": args.lr,
           "timing": "CUDA events around the whole scheduled epoch (training, swaps, test-loss evaluations)"}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    # default: the largest single-GPU configuration (Terabyte-shaped, RMC3)
    ap.add_argument("--config", default="terabyte", choices=sorted(gen.CONFIGS))
    ap.add_argument("--records", type=int, default=0, help="records per GPU (default: config)")
    ap.add_argument("--batch", type=int, default=0, help="hot mini-batch size B (default: config; batch sweeps)")
    ap.add_argument("--impl", default="fae", choices=["fae", "reference"])
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-records", type=int, default=0, help="cpu_baseline sample records (default per config)")
    ap.add_argument("--cpu-batches", type=int, default=0, help="cpu_baseline hot batches (default per config)")
    ap.add_argument("--ref-records", type=int, default=1_000_000, help="--impl reference: records per step")
    ap.add_argument("--ref-batches", type=int, default=16, help="--impl reference: hot batches per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ktiming", action="store_true", help="no in-kernel stamps (overhead check; no roofline)")
    ap.add_argument("--dy-pool-mb", type=int, default=256, help="upstream-gradient pool (> L2 by default)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--overlap", action="store_true",
                    help="A/B: step k+1's preprocessing on a second ctx / stream during step k's training "
                         "(measured slower on B200: the streaming preprocessing slows the latency-bound training)")
    ap.add_argument("--exchange", action="store_true",
                    help="N=1: run the multi-rank exchange loop on a 1-rank NCCL communicator (sync cost)")
    ap.add_argument("--sweep", action="store_true", help="threshold sweep (one JSON line; not the driver's bench)")
    ap.add_argument("--mixed", action="store_true", help="NEXT-1 timed mixed hot/cold epoch (one JSON line)")
    ap.add_argument("--rate", type=float, default=50.0, help="--mixed / --train: phase size (start), %% of each kind's batches")
    ap.add_argument("--train", action="store_true", help="NEXT-2/3: one scheduled FAE epoch of the paper's DLRM (one JSON line)")
    ap.add_argument("--lr-mlp", type=float, default=0.05)
    ap.add_argument("--test-records", type=int, default=65536)
    ap.add_argument("--sweep-configs", default="kaggle,terabyte")
    ap.add_argument("--sweep-fracs", default="1,2,5,10,20")
    args = ap.parse_args()
    if args.sweep:
        run_sweep(args)
        return
    if args.mixed:
        run_mixed(args)
        return
    if args.train:
        run_train(args)
        return
    if args.impl == "reference":
        r = run_reference(args)
        if r is not None:
            print(json.dumps(r), flush=True)
        return
    res, ctxs = run_fae(args)
    if not args.no_e2e:
        e2e = run_e2e(args, ctxs)
        if res is not None:
            res["e2e"] = e2e
    rank = int(os.environ.get("RANK", "0"))
    if rank == 0:
        cfg = gen.CONFIGS[args.config]
        if not args.no_cpu and res["n_gpus"] == 1:
            res["cpu_baseline"] = cpu_baseline(cfg, args)
        print(json.dumps(res), flush=True)
    dist = ctxs[5]
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
