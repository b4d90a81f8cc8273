"""CPU ORACLE for the FAE hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product path
(paper_2103_00686_b200) never imports it, and it imports nothing from the
product path.  The arithmetic lives in fae_oracle.c (plain C, fp64, written
from PAPER.md; see the citations there); this module only compiles it with
gcc and marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fae_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_fae.so")
_LIB_OMP = os.path.join(_HERE, "liboracle_fae_omp.so")   # the same file, -fopenmp
_lib = None
_lib_omp = None
_use_omp = False

OK, INVALID_ARG, BUDGET_INFEASIBLE, INDEX_RANGE = 0, 1, 3, 4


def build(force: bool = False) -> str:
    for out, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(out) or \
                os.path.getmtime(out) < os.path.getmtime(_SRC):
            subprocess.check_call(
                ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared", *extra,
                 "-o", out, _SRC, "-lm"])
    return _LIB


def use_omp(flag: bool) -> None:
    """Route the calls below to the all-cores build (-fopenmp; bit-identical
    results, tests/test_oracle.py) or back to the serial one."""
    global _use_omp
    _use_omp = bool(flag)


def omp_threads() -> int:
    """Threads the all-cores build uses (OMP_NUM_THREADS or all cores)."""
    n = os.environ.get("OMP_NUM_THREADS")
    return int(n) if n else (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())


def lib():
    global _lib, _lib_omp
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        _declare(_lib)
    if _use_omp:
        if _lib_omp is None:
            _lib_omp = ctypes.CDLL(_LIB_OMP)
            _declare(_lib_omp)
        return _lib_omp
    return _lib


P = ctypes.c_void_p
i32, i64, u64, f64, f32 = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                           ctypes.c_double, ctypes.c_float)


def _declare(L):
    L.or_mix64.restype = u64; L.or_mix64.argtypes = [u64]
    L.or_key.restype = u64; L.or_key.argtypes = [u64, u64]
    L.or_sample_count.restype = i64; L.or_sample_count.argtypes = [i64, f64]
    L.or_sample.restype = i64; L.or_sample.argtypes = [i64, f64, u64, P]
    L.or_histogram.restype = ctypes.c_int
    L.or_histogram.argtypes = [i32, P, P, P, i32, i64, P, i64, P, P]
    L.or_cutoff.restype = f64; L.or_cutoff.argtypes = [f64, i64, f64]
    L.or_kmin_from_cutoff.restype = i64; L.or_kmin_from_cutoff.argtypes = [f64]
    L.or_tag_rows.restype = None
    L.or_tag_rows.argtypes = [i32, P, i32, i64, P, P, P]
    L.or_kmin_fixed_t.restype = None
    L.or_kmin_fixed_t.argtypes = [i32, P, i32, i64, P, f64, f64, P]
    L.or_budget_exact.restype = ctypes.c_int
    L.or_budget_exact.argtypes = [i32, P, i32, i64, P, P, f64, i64, P, P, P, P]
    L.or_hot_bytes.restype = i64
    L.or_hot_bytes.argtypes = [i32, P, i32, i64, P, P]
    L.or_estimate.restype = None
    L.or_estimate.argtypes = [P, i64, i64, i32, i32, u64, f64, P, P, P]
    L.or_clt_search.restype = ctypes.c_int
    L.or_clt_search.argtypes = [i32, P, i32, i64, P, P, f64, i64, i32, i32, u64, f64, P, P, P, P, P]
    L.or_remap.restype = i64; L.or_remap.argtypes = [i32, P, P, P, P]
    L.or_classify.restype = None
    L.or_classify.argtypes = [i32, P, P, P, i32, i64, P, P]
    L.or_pack.restype = None
    L.or_pack.argtypes = [i32, P, P, P, i32, i64, P, P, P, P, P, P, P]
    L.or_extract.restype = None; L.or_extract.argtypes = [i64, i32, P, P, P]
    L.or_scatter_hot.restype = None; L.or_scatter_hot.argtypes = [i64, i32, P, P, P]
    L.or_emb_fwd.restype = ctypes.c_int
    L.or_emb_fwd.argtypes = [P, i64, i32, P, P, i32, i64, P]
    L.or_emb_bwd_sgd.restype = ctypes.c_int
    L.or_emb_bwd_sgd.argtypes = [P, i64, i32, P, P, i32, i64, P, f32, P]
    L.or_emb_grad.restype = i64
    L.or_emb_grad.argtypes = [i64, i32, P, P, i32, i64, P, P, P]


def _np(a, dtype):
    """torch tensor / list / ndarray -> C-contiguous ndarray of dtype."""
    if a is None:
        return None
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(P)


# --------------------------------------------------------------------------
def key(seed: int, i: int) -> int:
    return int(lib().or_key(seed, i))


def sample(R: int, x_pct: float, seed: int) -> np.ndarray:
    k = lib().or_sample_count(R, x_pct)
    if k < 0:
        raise ValueError("x must be in (0, 100]")
    out = np.empty(max(k, 1), np.int64)
    lib().or_sample(R, x_pct, seed, _ptr(out))
    return out[:k]


def histogram(rows, idx, off, fixed_pool, n_records, sampled):
    rows = _np(rows, np.int64)
    idx = _np(idx, np.int32)
    off = _np(off, np.int64)
    sampled = _np(sampled, np.int64)
    counts = np.zeros(int(rows.sum()), np.uint32)
    T = np.zeros(len(rows), np.int64)
    st = lib().or_histogram(len(rows), _ptr(rows), _ptr(idx), _ptr(off),
                            fixed_pool, n_records, _ptr(sampled), len(sampled),
                            _ptr(counts), _ptr(T))
    return counts, T, st


def cutoff(t: float, T: int, x_pct: float) -> float:
    return float(lib().or_cutoff(t, T, x_pct))


def kmin_from_cutoff(H: float) -> int:
    return int(lib().or_kmin_from_cutoff(H))


def kmin_fixed_t(rows, dim, small_bytes, T, t, x_pct):
    rows = _np(rows, np.int64); T = _np(T, np.int64)
    kmin = np.zeros(len(rows), np.int64)
    lib().or_kmin_fixed_t(len(rows), _ptr(rows), dim, small_bytes, _ptr(T),
                          t, x_pct, _ptr(kmin))
    return kmin


def tag_rows(rows, dim, small_bytes, counts, kmin):
    rows = _np(rows, np.int64); counts = _np(counts, np.uint32)
    kmin = _np(kmin, np.int64)
    hot = np.zeros(int(rows.sum()), np.uint8)
    lib().or_tag_rows(len(rows), _ptr(rows), dim, small_bytes, _ptr(counts),
                      _ptr(kmin), _ptr(hot))
    return hot


def budget_exact(rows, dim, small_bytes, counts, T, x_pct, budget_bytes):
    rows = _np(rows, np.int64); counts = _np(counts, np.uint32)
    T = _np(T, np.int64)
    kmin = np.zeros(len(rows), np.int64)
    K = ctypes.c_uint64(0); tf = ctypes.c_double(0); slack = ctypes.c_int32(0)
    st = lib().or_budget_exact(len(rows), _ptr(rows), dim, small_bytes,
                               _ptr(counts), _ptr(T), x_pct, budget_bytes,
                               _ptr(kmin), ctypes.byref(K), ctypes.byref(tf),
                               ctypes.byref(slack))
    return dict(status=st, kmin=kmin, K=K.value, t_final=tf.value,
                slack=slack.value)


def hot_bytes(rows, dim, small_bytes, counts, kmin) -> int:
    rows = _np(rows, np.int64); counts = _np(counts, np.uint32)
    kmin = _np(kmin, np.int64)
    return int(lib().or_hot_bytes(len(rows), _ptr(rows), dim, small_bytes,
                                  _ptr(counts), _ptr(kmin)))


def estimate(k_table, kmin, n=35, m=1024, chunk_seed=0, t_q=3.6007):
    k_table = _np(k_table, np.uint32)
    out = np.zeros(6, np.float64)
    C = np.zeros(n, np.int64); ch = np.zeros(n, np.int64)
    lib().or_estimate(_ptr(k_table), len(k_table), kmin, n, m, chunk_seed,
                      t_q, _ptr(out), _ptr(C), _ptr(ch))
    return dict(ybar=out[0], s=out[1], lo=out[2], hi=out[3], est=out[4],
                exact=bool(out[5]), C=C, chunks=ch)


def clt_search(rows, dim, small_bytes, counts, T, x_pct, budget_bytes, n=35, m=1024,
               chunk_seed=0, t_q=3.6007):
    """CLT-driven statistical optimizer (or_clt_search, R27)."""
    rows = _np(rows, np.int64); counts = _np(counts, np.uint32)
    T = _np(T, np.int64)
    kmin = np.zeros(len(rows), np.int64)
    tf = ctypes.c_double(0); bf = ctypes.c_double(0)
    slack = ctypes.c_int32(0); ev = ctypes.c_int32(0)
    st = lib().or_clt_search(len(rows), _ptr(rows), dim, small_bytes, _ptr(counts), _ptr(T),
                             x_pct, budget_bytes, n, m, chunk_seed, t_q, _ptr(kmin),
                             ctypes.byref(tf), ctypes.byref(bf), ctypes.byref(slack),
                             ctypes.byref(ev))
    return dict(status=st, kmin=kmin, t_final=tf.value, est_bytes=bf.value,
                slack=slack.value, evals=ev.value)


def remap(rows, hot):
    rows = _np(rows, np.int64); hot = _np(hot, np.uint8)
    rm = np.empty(int(rows.sum()), np.int32)
    base = np.zeros(len(rows) + 1, np.int64)
    H = lib().or_remap(len(rows), _ptr(rows), _ptr(hot), _ptr(rm), _ptr(base))
    return rm, base, int(H)


def classify(rows, idx, off, fixed_pool, n_records, remap_):
    rows = _np(rows, np.int64); idx = _np(idx, np.int32)
    off = _np(off, np.int64); remap_ = _np(remap_, np.int32)
    flag = np.zeros(n_records, np.uint8)
    lib().or_classify(len(rows), _ptr(rows), _ptr(idx), _ptr(off), fixed_pool,
                      n_records, _ptr(remap_), _ptr(flag))
    return flag


def pack(rows, idx, off, fixed_pool, n_records, remap_, flag):
    rows = _np(rows, np.int64); idx = _np(idx, np.int32)
    off = _np(off, np.int64); remap_ = _np(remap_, np.int32)
    flag = _np(flag, np.uint8)
    n_hot = int(flag.sum())
    Tn = len(rows)
    hot_ids = np.empty(max(n_hot, 1), np.int64)
    cold_ids = np.empty(max(n_records - n_hot, 1), np.int64)
    hot_idx = np.empty(max(len(idx), 1), np.int32)
    hot_off = np.empty(n_hot * Tn + 1, np.int64) if off is not None else None
    cnt = np.zeros(3, np.int64)
    lib().or_pack(Tn, _ptr(rows), _ptr(idx), _ptr(off), fixed_pool, n_records,
                  _ptr(remap_), _ptr(flag), _ptr(hot_ids), _ptr(cold_ids),
                  _ptr(hot_idx), _ptr(hot_off), _ptr(cnt))
    nh, nc, nl = (int(v) for v in cnt)
    return dict(hot_ids=hot_ids[:nh], cold_ids=cold_ids[:nc],
                hot_idx=hot_idx[:nl], hot_off=hot_off, n_hot=nh, n_cold=nc,
                n_hot_lookups=nl)


def extract(W, remap_, H):
    W = _np(W, np.float32); remap_ = _np(remap_, np.int32)
    dim = W.shape[1]
    out = np.zeros((max(H, 1), dim), np.float32)
    lib().or_extract(W.shape[0], dim, _ptr(W), _ptr(remap_), _ptr(out))
    return out[:H]


def scatter_hot(W, W_hot, remap_):
    """NEXT-1 swap sync: a copy of W with W[g] = W_hot[remap[g]] for hot g."""
    W = _np(W, np.float32).copy(); W_hot = _np(W_hot, np.float32)
    remap_ = _np(remap_, np.int32)
    lib().or_scatter_hot(W.shape[0], W.shape[1], _ptr(W_hot), _ptr(remap_), _ptr(W))
    return W


def emb_fwd(W_hot, idx, off, fixed_pool, n_bags):
    W_hot = _np(W_hot, np.float32); idx = _np(idx, np.int32)
    off = _np(off, np.int64)
    dim = W_hot.shape[1]
    Y = np.zeros((n_bags, dim), np.float32)
    st = lib().or_emb_fwd(_ptr(W_hot), W_hot.shape[0], dim, _ptr(idx),
                          _ptr(off), fixed_pool, n_bags, _ptr(Y))
    return Y, st


def emb_bwd_sgd(W_hot, idx, off, fixed_pool, n_bags, dY, lr,
                slot: Optional[np.ndarray] = None):
    """Returns the updated copy of W_hot (the input is not modified)."""
    W = _np(W_hot, np.float32).copy()
    idx = _np(idx, np.int32); off = _np(off, np.int64)
    dY = _np(dY, np.float32)
    if slot is None:
        slot = np.full(W.shape[0], -1, np.int32)
    st = lib().or_emb_bwd_sgd(_ptr(W), W.shape[0], W.shape[1], _ptr(idx),
                              _ptr(off), fixed_pool, n_bags, _ptr(dY),
                              ctypes.c_float(lr), _ptr(slot))
    return W, st


def emb_grad(H, dim, idx, off, fixed_pool, n_bags, dY):
    idx = _np(idx, np.int32); off = _np(off, np.int64)
    dY = _np(dY, np.float32)
    L = len(idx)
    rows_out = np.empty(max(L, 1), np.int32)
    G = np.zeros((max(L, 1), dim), np.float64)
    U = lib().or_emb_grad(H, dim, _ptr(idx), _ptr(off), fixed_pool, n_bags,
                          _ptr(dY), _ptr(rows_out), _ptr(G))
    return rows_out[:U], G[:U]
