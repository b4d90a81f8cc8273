"""B200-native FAE hot path — thin Python binding of libfae.so (include/fae.h).

Argument marshalling only: every step of the path runs in the CUDA kernels of
libfae.so.  PyTorch supplies device memory (tensor data pointers) and the
stream.  There is no CPU fallback: if the library is missing or a call fails,
an exception is raised.

Names follow the C ABI (fae_profile, fae_threshold, fae_classify, fae_extract,
fae_emb_fwd, fae_emb_bwd_update, fae_sync_hot_grads).  See include/fae.h for
argument meaning, layout, ownership and errors, with PAPER.md citations.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FAE_LIB: load another build of the same ABI (A/B timing of two builds)
LIB_PATH = os.environ.get("FAE_LIB") or os.path.join(_HERE, "_lib", "libfae.so")
_lib = None

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "CAPACITY", 3: "BUDGET_INFEASIBLE",
          4: "INDEX_RANGE", 5: "NONFINITE", 6: "CUDA", 7: "NCCL", 8: "NOT_INIT"}
FIXED_T, BUDGET_EXACT, CLT_SEARCH = 0, 1, 2

EXPORTS = ["fae_create", "fae_destroy", "fae_set_stream", "fae_last_error",
           "fae_check", "fae_get_nccl_id", "fae_comm_init", "fae_comm_init_loopback",
           "fae_kernel_launches", "fae_profile", "fae_threshold",
           "fae_classify", "fae_extract", "fae_scatter_hot", "fae_pack_cold", "fae_emb_fwd", "fae_emb_bwd_update",
           "fae_sync_hot_grads", "fae_group_batches", "fae_release_scratch", "fae_train_hot_batches",
           "fae_set_kernel_timing", "fae_get_kernel_timing", "fae_get_exchange_timing", "fae_group_info",
           "fae_sched_init", "fae_sched_next", "fae_sched_record_swap", "fae_sched_new_epoch",
           "fae_dlrm_param_count", "fae_dlrm_create", "fae_dlrm_destroy", "fae_dlrm_step", "fae_dlrm_loss",
           "fae_dlrm_buffers", "fae_train_dlrm_batches"]


SCHED_MAX_U = 64


class FaeSched(ctypes.Structure):
    """fae_sched (include/fae.h): the scheduler's plain state (NEXT-3)."""
    _fields_ = [("n", ctypes.c_int64 * 2), ("done", ctypes.c_int64 * 2), ("r", ctypes.c_double),
                ("u", ctypes.c_int32), ("next_kind", ctypes.c_int32), ("last_kind", ctypes.c_int32),
                ("n_hist", ctypes.c_int32), ("hist", ctypes.c_double * (SCHED_MAX_U + 1)),
                ("swaps", ctypes.c_int64), ("sync_events", ctypes.c_int64), ("sync_bytes", ctypes.c_int64)]


DLRM_MAX_LAYERS = 8


class FaeDlrmCfg(ctypes.Structure):
    """fae_dlrm_cfg (include/fae.h, NEXT-2)."""
    _fields_ = [("n_dense", ctypes.c_int32), ("n_bottom", ctypes.c_int32),
                ("bottom", ctypes.c_int32 * DLRM_MAX_LAYERS), ("n_top", ctypes.c_int32),
                ("top", ctypes.c_int32 * DLRM_MAX_LAYERS), ("n_tables", ctypes.c_int32),
                ("dim", ctypes.c_int32), ("max_batch", ctypes.c_int32), ("tf32", ctypes.c_int32)]


class FaeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


c_i32, c_i64, c_u64, c_dbl, c_ptr = (ctypes.c_int32, ctypes.c_int64,
                                     ctypes.c_uint64, ctypes.c_double,
                                     ctypes.c_void_p)


class FaeConfig(ctypes.Structure):
    _fields_ = [("device", c_i32), ("max_tables", c_i32), ("max_rows", c_i64),
                ("max_batch_lookups", c_i64), ("max_batch_bags", c_i64),
                ("max_dim", c_i32), ("max_world", c_i32)]


class FaeTables(ctypes.Structure):
    _fields_ = [("n_tables", c_i32), ("rows", c_ptr), ("dim", c_i32)]


class FaeCsr(ctypes.Structure):
    _fields_ = [("idx", c_ptr), ("off", c_ptr), ("fixed_pool", c_i32),
                ("n_records", c_i64), ("n_lookups", c_i64),
                ("record_base", c_i64), ("n_records_global", c_i64)]


class FaeThreshReq(ctypes.Structure):
    _fields_ = [("mode", c_i32), ("t", c_dbl), ("budget_bytes", c_i64),
                ("small_table_bytes", c_i64), ("want_estimate", c_i32),
                ("n_chunks", c_i32), ("chunk_rows", c_i32),
                ("t_quantile", c_dbl), ("chunk_seed", c_u64)]


class FaeThreshResult(ctypes.Structure):
    _fields_ = [("kmin", c_ptr), ("hot_rows", c_ptr), ("base", c_ptr),
                ("is_small", c_ptr), ("est_mean", c_ptr), ("est_sd", c_ptr),
                ("est_lo", c_ptr), ("est_hi", c_ptr), ("est_rows", c_ptr),
                ("est_exact", c_ptr), ("H_total", c_i64), ("hot_bytes", c_i64),
                ("t_final", c_dbl), ("K", c_u64), ("budget_slack", c_i32)]


class FaePacked(ctypes.Structure):
    _fields_ = [("hot_ids", c_ptr), ("cold_ids", c_ptr), ("hot_idx", c_ptr),
                ("hot_off", c_ptr), ("n_hot", c_i64), ("n_cold", c_i64),
                ("n_hot_lookups", c_i64), ("n_hot_batches", c_i64),
                ("n_cold_batches", c_i64)]


def lib():
    """Load libfae.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libfae.so not built ({LIB_PATH}); run "
                              "python -m paper_2103_00686_b200.build")
        L = ctypes.CDLL(LIB_PATH)
        P = c_ptr
        sig = {
            "fae_create": ([ctypes.POINTER(FaeConfig), ctypes.POINTER(c_ptr)], c_i32),
            "fae_destroy": ([P], None),
            "fae_set_stream": ([P, P], c_i32),
            "fae_last_error": ([P], ctypes.c_char_p),
            "fae_check": ([P], c_i32),
            "fae_get_nccl_id": ([P], c_i32),
            "fae_comm_init": ([P, P, c_i32, c_i32], c_i32),
            "fae_comm_init_loopback": ([P, c_u64, c_i32, c_i32], c_i32),
            "fae_kernel_launches": ([P], c_i64),
            "fae_profile": ([P, ctypes.POINTER(FaeTables), ctypes.POINTER(FaeCsr),
                             c_dbl, c_u64, P, P, P, P], c_i32),
            "fae_threshold": ([P, ctypes.POINTER(FaeTables), P, P, c_dbl,
                               ctypes.POINTER(FaeThreshReq), P,
                               ctypes.POINTER(FaeThreshResult)], c_i32),
            "fae_classify": ([P, ctypes.POINTER(FaeTables), ctypes.POINTER(FaeCsr),
                              c_i32, c_u64, ctypes.POINTER(FaePacked)], c_i32),
            "fae_extract": ([P, P, c_i32, P], c_i32),
            "fae_scatter_hot": ([P, P, c_i32, P], c_i32),
            "fae_pack_cold": ([P, ctypes.POINTER(FaeTables), ctypes.POINTER(FaeCsr), P, c_i64, P, P], c_i32),
            "fae_emb_fwd": ([P, P, c_i64, c_i32, P, P, c_i32, c_i64, P], c_i32),
            "fae_emb_bwd_update": ([P, P, c_i64, c_i32, P, P, c_i32, c_i64, P,
                                    ctypes.c_float], c_i32),
            "fae_sync_hot_grads": ([P, P, P, P, c_i64, c_i32], c_i32),
            "fae_group_batches": ([P, ctypes.POINTER(FaeTables), ctypes.POINTER(FaePacked),
                                   c_i32, c_i32, c_i64], c_i32),
            "fae_release_scratch": ([P], c_i32),
            "fae_train_hot_batches": ([P, P, c_i64, c_i32, c_i64, c_i64, P, c_i64, P,
                                       ctypes.c_float], c_i32),
            "fae_set_kernel_timing": ([P, c_i32], c_i32),
            "fae_get_kernel_timing": ([P, P, P], c_i32),
            "fae_get_exchange_timing": ([P, P], c_i32),
            "fae_group_info": ([P, P], c_i32),
            "fae_sched_init": ([ctypes.POINTER(FaeSched), c_i64, c_i64, c_dbl, c_i32], c_i32),
            "fae_sched_next": ([ctypes.POINTER(FaeSched), P, P, P, P], c_i32),
            "fae_sched_record_swap": ([ctypes.POINTER(FaeSched), c_dbl, c_i64, c_i32], c_i32),
            "fae_sched_new_epoch": ([ctypes.POINTER(FaeSched)], c_i32),
            "fae_dlrm_param_count": ([ctypes.POINTER(FaeDlrmCfg)], c_i64),
            "fae_dlrm_create": ([P, ctypes.POINTER(FaeDlrmCfg), P], c_i32),
            "fae_dlrm_destroy": ([P], None),
            "fae_dlrm_step": ([P, P, c_i32, P, P, P, P, ctypes.c_float, c_i32], c_i32),
            "fae_dlrm_loss": ([P, P, P, c_i32], c_i32),
            "fae_dlrm_buffers": ([P, P, P, P], c_i32),
            "fae_train_dlrm_batches": ([P, P, P, P, c_i64, c_i32, c_i64, c_i64, P, P, P, ctypes.c_float,
                                        ctypes.c_float], c_i32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _p(t: Optional[torch.Tensor]):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


class Ctx:
    """Owns one fae_ctx (one per GPU / rank)."""

    def __init__(self, handle, device: int):
        self.h = handle
        self.device = device

    def close(self):
        if self.h:
            lib().fae_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ok(self, st: int):
        if st != 0:
            msg = lib().fae_last_error(self.h) or b""
            raise FaeError(st, msg.decode(errors="replace"))

    def set_stream(self, stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._ok(lib().fae_set_stream(self.h, ctypes.c_void_p(s.cuda_stream)))

    def check(self):
        self._ok(lib().fae_check(self.h))

    @property
    def launches(self) -> int:
        return int(lib().fae_kernel_launches(self.h))


def fae_create(device: int = 0, max_tables: int = 64, max_rows: int = 1 << 20,
               max_batch_lookups: int = 1 << 20, max_batch_bags: int = 1 << 20,
               max_dim: int = 128, max_world: int = 1) -> Ctx:
    cfg = FaeConfig(device, max_tables, max_rows, max_batch_lookups,
                    max_batch_bags, max_dim, max_world)
    h = c_ptr()
    st = lib().fae_create(ctypes.byref(cfg), ctypes.byref(h))
    if st != 0:
        raise FaeError(st, "fae_create failed")
    ctx = Ctx(h, device)
    ctx.set_stream()
    return ctx


def fae_get_nccl_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = lib().fae_get_nccl_id(buf)
    if st != 0:
        raise FaeError(st, "ncclGetUniqueId failed")
    return buf.raw


def fae_comm_init(ctx: Ctx, nccl_id: bytes, rank: int, world: int):
    buf = ctypes.create_string_buffer(nccl_id, 128)
    ctx._ok(lib().fae_comm_init(ctx.h, buf, rank, world))


def fae_comm_init_loopback(ctx: Ctx, group_key: int, rank: int, world: int):
    """TEST-ONLY virtual ranks on one GPU (needs FAE_LOOPBACK=1); see fae.h."""
    ctx._ok(lib().fae_comm_init_loopback(ctx.h, ctypes.c_uint64(group_key), rank, world))


def _tables(rows: Sequence[int], dim: int):
    arr = (c_i64 * len(rows))(*[int(r) for r in rows])
    return FaeTables(len(rows), ctypes.cast(arr, c_ptr), dim), arr


def _csr(idx: torch.Tensor, off: Optional[torch.Tensor], fixed_pool: int,
         n_records: int, n_tables: int, record_base: int = 0,
         n_records_global: Optional[int] = None) -> FaeCsr:
    n_lookups = int(idx.numel())
    if off is not None:
        assert off.dtype == torch.int64 and off.is_contiguous()
    assert idx.dtype == torch.int32 and idx.is_contiguous()
    return FaeCsr(_p(idx) if n_lookups else None, _p(off), int(fixed_pool),
                  int(n_records), n_lookups, int(record_base),
                  int(n_records if n_records_global is None else n_records_global))


def fae_profile(ctx: Ctx, rows, dim: int, idx, off, fixed_pool: int,
                n_records: int, x_pct: float, seed: int, counts: torch.Tensor,
                sampled_ids: Optional[torch.Tensor] = None,
                record_base: int = 0, n_records_global: Optional[int] = None):
    """a1 + a2.  Returns (T list, n_sampled)."""
    tabs, keep = _tables(rows, dim)
    csr = _csr(idx, off, fixed_pool, n_records, len(rows), record_base,
               n_records_global)
    T = (c_i64 * len(rows))()
    ns = c_i64(0)
    ctx._ok(lib().fae_profile(ctx.h, ctypes.byref(tabs), ctypes.byref(csr),
                              float(x_pct), ctypes.c_uint64(seed & (2**64 - 1)),
                              _p(counts), ctypes.cast(T, c_ptr), _p(sampled_ids),
                              ctypes.byref(ns)))
    del keep
    return [int(v) for v in T], int(ns.value)


def fae_threshold(ctx: Ctx, rows, dim: int, counts: torch.Tensor, T, x_pct: float,
                  mode: int = FIXED_T, t: float = 0.0, budget_bytes: int = 0,
                  small_table_bytes: int = 1 << 20, want_estimate: bool = False,
                  n_chunks: int = 35, chunk_rows: int = 1024,
                  t_quantile: float = 3.6007, chunk_seed: int = 0,
                  remap_out: Optional[torch.Tensor] = None) -> dict:
    """a3 + a4.  Returns the fae_thresh_result fields as a dict."""
    tabs, keep = _tables(rows, dim)
    n = len(rows)
    Th = (c_i64 * n)(*[int(v) for v in T])
    req = FaeThreshReq(mode, float(t), int(budget_bytes), int(small_table_bytes),
                       int(bool(want_estimate)), n_chunks, chunk_rows,
                       float(t_quantile), chunk_seed & (2**64 - 1))
    arrs = {k: (c_i64 * n)() for k in ("kmin", "hot_rows")}
    arrs["base"] = (c_i64 * (n + 1))()
    arrs["is_small"] = (c_i32 * n)()
    for k in ("est_mean", "est_sd", "est_lo", "est_hi", "est_rows"):
        arrs[k] = (c_dbl * n)()
    arrs["est_exact"] = (c_i32 * n)()
    res = FaeThreshResult(**{k: ctypes.cast(v, c_ptr) for k, v in arrs.items()})
    ctx._ok(lib().fae_threshold(ctx.h, ctypes.byref(tabs), _p(counts),
                                ctypes.cast(Th, c_ptr), float(x_pct),
                                ctypes.byref(req), _p(remap_out),
                                ctypes.byref(res)))
    del keep
    out = {k: list(v) for k, v in arrs.items()}
    out.update(H_total=res.H_total, hot_bytes=res.hot_bytes,
               t_final=res.t_final, K=res.K, budget_slack=res.budget_slack)
    return out


def fae_classify(ctx: Ctx, rows, dim: int, idx, off, fixed_pool: int,
                 n_records: int, batch: int, hot_ids: torch.Tensor,
                 cold_ids: torch.Tensor, hot_idx: torch.Tensor,
                 hot_off: Optional[torch.Tensor] = None,
                 shuffle_seed: int = 0) -> dict:
    """a5 + a6.  Returns counts (n_hot, n_cold, n_hot_lookups, batches)."""
    tabs, keep = _tables(rows, dim)
    csr = _csr(idx, off, fixed_pool, n_records, len(rows))
    pk = FaePacked(_p(hot_ids), _p(cold_ids), _p(hot_idx), _p(hot_off))
    ctx._ok(lib().fae_classify(ctx.h, ctypes.byref(tabs), ctypes.byref(csr),
                               int(batch), ctypes.c_uint64(shuffle_seed),
                               ctypes.byref(pk)))
    del keep
    return dict(n_hot=pk.n_hot, n_cold=pk.n_cold, n_hot_lookups=pk.n_hot_lookups,
                n_hot_batches=pk.n_hot_batches, n_cold_batches=pk.n_cold_batches)


def fae_extract(ctx: Ctx, W: torch.Tensor, W_hot: torch.Tensor):
    """a7: W may be a CUDA tensor or a pinned CPU tensor (mapped)."""
    assert W.dtype == torch.float32 and W.is_contiguous()
    ctx._ok(lib().fae_extract(ctx.h, _p(W), int(W.shape[1]), _p(W_hot)))


def fae_scatter_hot(ctx: Ctx, W_hot: torch.Tensor, W: torch.Tensor):
    """NEXT-1 swap sync: W[g] = W_hot[hot_id(g)] for hot rows (inverse of
    fae_extract); W may be a CUDA tensor or a pinned CPU tensor (mapped)."""
    assert W.dtype == torch.float32 and W.is_contiguous()
    ctx._ok(lib().fae_scatter_hot(ctx.h, _p(W_hot), int(W.shape[1]), _p(W)))


def fae_pack_cold(ctx: Ctx, rows, dim: int, idx: torch.Tensor, fixed_pool: int, n_records: int,
                  cold_ids: torch.Tensor, n_cold: int, cold_idx: torch.Tensor,
                  off: Optional[torch.Tensor] = None, cold_off: Optional[torch.Tensor] = None):
    """NEXT-1 cold side: the cold records' lookups in global row ids
    (cold_off: their bag offsets, explicit-offset inputs only)."""
    tabs, keep = _tables(rows, dim)
    csr = _csr(idx, off, fixed_pool, n_records, len(rows))
    ctx._ok(lib().fae_pack_cold(ctx.h, ctypes.byref(tabs), ctypes.byref(csr), _p(cold_ids),
                                int(n_cold), _p(cold_idx), _p(cold_off)))
    del keep


def fae_emb_fwd(ctx: Ctx, W_hot: torch.Tensor, idx: torch.Tensor,
                off: Optional[torch.Tensor], fixed_pool: int, n_bags: int,
                Y: torch.Tensor):
    """a8: Y[b] = sum of W_hot rows of bag b (sum pooling)."""
    ctx._ok(lib().fae_emb_fwd(ctx.h, _p(W_hot), int(W_hot.shape[0]),
                              int(W_hot.shape[1]), _p(idx), _p(off),
                              int(fixed_pool), int(n_bags), _p(Y)))


def fae_emb_bwd_update(ctx: Ctx, W_hot: torch.Tensor, idx: torch.Tensor,
                       off: Optional[torch.Tensor], fixed_pool: int,
                       n_bags: int, dY: torch.Tensor, lr: float):
    """a9 + a10 (+ a11 with a comm): W_hot[r] -= lr * sum of dY rows of r."""
    ctx._ok(lib().fae_emb_bwd_update(ctx.h, _p(W_hot), int(W_hot.shape[0]),
                                     int(W_hot.shape[1]), _p(idx), _p(off),
                                     int(fixed_pool), int(n_bags), _p(dY),
                                     ctypes.c_float(lr)))


def fae_sync_hot_grads(ctx: Ctx, rows: torch.Tensor, vals: torch.Tensor,
                       count: int) -> int:
    """a11 on a caller-visible sparse gradient; returns the global count."""
    cnt = c_i64(int(count))
    ctx._ok(lib().fae_sync_hot_grads(ctx.h, _p(rows), _p(vals), ctypes.byref(cnt),
                                     int(rows.numel()), int(vals.shape[1])))
    return int(cnt.value)


def fae_group_batches(ctx: Ctx, rows, dim: int, hot_idx: torch.Tensor,
                      hot_off: Optional[torch.Tensor], n_hot: int,
                      n_hot_lookups: int, fixed_pool: int, batch: int, H: int):
    """a9's sort-and-segment for every hot batch, once (kept in the ctx;
    hot_idx / hot_off must stay alive and unchanged)."""
    tabs, keep = _tables(rows, dim)
    pk = FaePacked(_p(hot_idx), None, _p(hot_idx), _p(hot_off), int(n_hot), 0,
                   int(n_hot_lookups), 0, 0)
    ctx._ok(lib().fae_group_batches(ctx.h, ctypes.byref(tabs), ctypes.byref(pk),
                                    int(fixed_pool), int(batch), int(H)))
    del keep


def fae_release_scratch(ctx: Ctx):
    """Free the last grouping's build-only scratch (kept: what training reads)."""
    ctx._ok(lib().fae_release_scratch(ctx.h))


def fae_train_hot_batches(ctx: Ctx, W_hot: torch.Tensor, first: int, n: int,
                          dY: torch.Tensor, Y: torch.Tensor, lr: float):
    """a8-a10 (+a11) over grouped hot batches [first, first+n); dY is
    [n_dy, B*Tn, D] (batch i uses dY[i % n_dy]), Y is [B*Tn, D]."""
    n_dy = int(dY.shape[0]) if dY.dim() == 3 else 1
    ctx._ok(lib().fae_train_hot_batches(ctx.h, _p(W_hot), int(W_hot.shape[0]),
                                        int(W_hot.shape[1]), int(first), int(n),
                                        _p(dY), n_dy, _p(Y), ctypes.c_float(lr)))


def fae_set_kernel_timing(ctx: Ctx, mode: int):
    """0 off; 1 in-kernel globaltimer stamps (keeps the PDL overlap; each
    kernel's exclusive share of the step); 2 CUDA event nodes in the graph
    (serialises the kernels; cross-check)."""
    ctx._ok(lib().fae_set_kernel_timing(ctx.h, int(mode)))


def fae_get_kernel_timing(ctx: Ctx) -> dict:
    """{'fwd': (total_ms, launches), 'reduce': (total_ms, launches), ...};
    mode 'persist': 'reduce' holds the persistent epoch kernel's (total_ms,
    launches) and 'persist_batches' the batches those launches trained."""
    ms = (c_dbl * 4)()
    n = (c_i64 * 4)()
    ctx._ok(lib().fae_get_kernel_timing(ctx.h, ctypes.cast(ms, c_ptr), ctypes.cast(n, c_ptr)))
    return {"fwd": (ms[0], n[0]), "reduce": (ms[1], n[1]),
            "overlap": (ms[2], n[2]), "fused": n[3] == 1, "persist": n[3] == 2,
            "persist_batches": int(ms[3])}


def fae_get_exchange_timing(ctx: Ctx) -> dict:
    """Exchange loop (world > 1): all-gather / merge ms summed over the timed
    steps, steps timed, slot bytes this rank contributed, steps run, and the
    last call's padded per-rank entries xcap."""
    out = (c_dbl * 6)()
    ctx._ok(lib().fae_get_exchange_timing(ctx.h, ctypes.cast(out, c_ptr)))
    return {"allgather_ms": out[0], "merge_ms": out[1], "steps_timed": int(out[2]),
            "slot_bytes": out[3], "steps": int(out[4]), "xcap": int(out[5])}


def fae_group_info(ctx: Ctx) -> dict:
    info = (c_i64 * 8)()
    ctx._ok(lib().fae_group_info(ctx.h, ctypes.cast(info, c_ptr)))
    keys = ("n_batches", "lookups", "long_segments", "segments", "max_long", "max_bags",
            "free_segments", "fused")
    return dict(zip(keys, [int(v) for v in info]))


# ---------------------------------------------------------------------------
# scheduler (NEXT-3, host-only; §4.3 Eq. 5)
# ---------------------------------------------------------------------------
class Scheduler:
    """Cold/hot phase interleaving with Eq. 5's loss-feedback rate
    (libfae's fae_sched_*; argument marshalling only)."""
    KINDS = ("cold", "hot")

    def __init__(self, n_cold: int, n_hot: int, r_start: float = 50.0, u: int = 4):
        self.s = FaeSched()
        st = lib().fae_sched_init(ctypes.byref(self.s), int(n_cold), int(n_hot), float(r_start), int(u))
        if st != 0:
            raise FaeError(st, "fae_sched_init: bad arguments")

    def next_phase(self):
        """(kind, first, count, swap_after) or None once both kinds are drained."""
        k, f, c, w = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        st = lib().fae_sched_next(ctypes.byref(self.s), ctypes.byref(k), ctypes.byref(f), ctypes.byref(c),
                                  ctypes.byref(w))
        if st != 0:
            raise FaeError(st, "fae_sched_next")
        if c.value == 0:
            return None
        return self.KINDS[k.value], int(f.value), int(c.value), bool(w.value)

    def record_swap(self, test_loss: float, hot_bytes: int = 0, n_devices: int = 1):
        st = lib().fae_sched_record_swap(ctypes.byref(self.s), float(test_loss), int(hot_bytes), int(n_devices))
        if st != 0:
            raise FaeError(st, "fae_sched_record_swap: bad arguments")

    def new_epoch(self):
        lib().fae_sched_new_epoch(ctypes.byref(self.s))

    @property
    def rate(self) -> float:
        return float(self.s.r)

    @property
    def swaps(self) -> int:
        return int(self.s.swaps)


# ---------------------------------------------------------------------------
# DLRM hot step (NEXT-2)
# ---------------------------------------------------------------------------
class Dlrm:
    """The DLRM of a hot mini-batch (libfae's fae_dlrm_*; marshalling only).
    Parameters live in one flat device fp32 tensor (per layer W [out][in],
    then b [out]; bottom layers first)."""

    def __init__(self, ctx: Ctx, n_dense: int, bottom, top, n_tables: int, dim: int,
                 max_batch: int, tf32: bool = True):
        cfg = FaeDlrmCfg()
        cfg.n_dense, cfg.n_bottom, cfg.n_top = int(n_dense), len(bottom), len(top)
        for i, w in enumerate(bottom):
            cfg.bottom[i] = int(w)
        for i, w in enumerate(top):
            cfg.top[i] = int(w)
        cfg.n_tables, cfg.dim, cfg.max_batch, cfg.tf32 = int(n_tables), int(dim), int(max_batch), int(bool(tf32))
        self.cfg, self.ctx = cfg, ctx
        self.n_params = int(lib().fae_dlrm_param_count(ctypes.byref(cfg)))
        if self.n_params < 0:
            raise FaeError(1, "fae_dlrm_param_count: invalid configuration")
        h = ctypes.c_void_p()
        ctx._ok(lib().fae_dlrm_create(ctx.h, ctypes.byref(cfg), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().fae_dlrm_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def step(self, params: torch.Tensor, B: int, dense, label, Y, dY=None, lr: float = 0.0,
             train: bool = True):
        self.ctx._ok(lib().fae_dlrm_step(self.h, _p(params), int(B), _p(dense), _p(label), _p(Y), _p(dY),
                                         ctypes.c_float(lr), int(bool(train))))

    def loss(self, reset: bool = True):
        """(sum of per-sample losses, samples) accumulated on the device."""
        a, b = ctypes.c_double(), ctypes.c_double()
        self.ctx._ok(lib().fae_dlrm_loss(self.h, ctypes.byref(a), ctypes.byref(b), int(bool(reset))))
        return a.value, b.value

    def buffers(self):
        """Device pointers (Y, dY, loss accumulator) of the model's batch buffers."""
        y, dy, acc = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        self.ctx._ok(lib().fae_dlrm_buffers(self.h, ctypes.byref(y), ctypes.byref(dy), ctypes.byref(acc)))
        return y.value, dy.value, acc.value

    def train_batches(self, params, W_hot, first: int, n: int, hot_ids, dense, label,
                      lr_mlp: float, lr_emb: float):
        """The full hot step over grouped hot batches [first, first + n)."""
        self.ctx._ok(lib().fae_train_dlrm_batches(self.ctx.h, self.h, _p(params), _p(W_hot),
                                                  int(W_hot.shape[0]), int(W_hot.shape[1]), int(first), int(n),
                                                  _p(hot_ids), _p(dense), _p(label), ctypes.c_float(lr_mlp),
                                                  ctypes.c_float(lr_emb)))
