"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no sampling rule, no
histogram, no threshold, no classification, no pooling, no gradient).  It only
draws the synthetic inputs the paper's workloads are shaped like:

* sparse inputs: per table z, a Zipf(s) rank rho over [1, N_z] mapped to a row
  by a seeded Feistel bijection pi_z (so hot rows are scattered, as in real
  data); sample-major CSR layout (record r, table z, pooling slot p);
* dense fp32 tensors: the full embedding tables W (U(-0.05, 0.05)) and the
  upstream gradients dY (U(-1, 1)).

Everything is a pure function of (seed, counter) through a splitmix64 counter
hash, evaluated with torch int64 ops so the same call gives the same bits on
CPU and on CUDA.  Shapes follow BASELINE.json "configs" and SURVEY.md §8(d);
the recipe is restated in DESIGN.md §"Input recipe".
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import torch

GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
BASE_SEED = 20260101


def _s64(v: int) -> int:
    """Python int -> the int64 with the same 64 low bits."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 tensors (torch's >> is arithmetic)."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def mix64(z: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (wrap-around arithmetic)."""
    z = z ^ _srl(z, 30)
    z = z * _s64(_M1)
    z = z ^ _srl(z, 27)
    z = z * _s64(_M2)
    z = z ^ _srl(z, 31)
    return z


def counter_hash(seed: int, ctr: torch.Tensor) -> torch.Tensor:
    """mix64(seed + (ctr + 1) * GOLDEN) for an int64 counter tensor."""
    return mix64((ctr + 1) * _s64(GOLDEN) + _s64(seed))


def uniform01(seed: int, ctr: torch.Tensor) -> torch.Tensor:
    """Exact dyadic uniforms in (0, 1): ((h >>> 11) + 0.5) / 2^53, fp64."""
    h = _srl(counter_hash(seed, ctr), 11)
    return (h.double() + 0.5) * (2.0 ** -53)


# ----------------------------------------------------------------------------
# Configurations (BASELINE.json "configs")
# ----------------------------------------------------------------------------
KAGGLE_ROWS = [1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145,
               5683, 8351593, 3194, 27, 14992, 5461306, 10, 5652, 2173, 4,
               7046547, 18, 15, 286181, 105, 142572]
TERABYTE_ROWS = [39884406, 39043, 17289, 7420, 20263, 3, 7120, 1543, 63,
                 38532951, 2953546, 403346, 10, 2208, 11938, 155, 4, 976, 14,
                 39979771, 25641295, 39664984, 585935, 12972, 108, 36]
ALIBABA_ROWS = [987994, 4162024, 9439]


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    rows: List[int]
    dim: int
    batch: int                 # per-GPU mini-batch (records), weak scaling
    pool: int                  # fixed pooling factor; 0 => variable (offsets)
    pool_lo: int = 0           # variable pooling range (inclusive)
    pool_hi: int = 0
    zipf_s: float = 1.1
    records: int = 0           # full dataset size R
    t: float = 1e-7            # default fixed threshold (fraction)
    budget_bytes: int = 0      # default hot budget (0 => FIXED_T)
    small_bytes: int = 1 << 20  # P:L386-387 small-table rule

    @property
    def n_tables(self) -> int:
        return len(self.rows)


CONFIGS = {
    "tiny": Config("tiny", [1000] * 4, 16, 128, 1, records=10_000, t=1e-2,
                   small_bytes=0),
    "kaggle": Config("kaggle", KAGGLE_ROWS, 16, 2048, 1, records=45_000_000,
                     t=1e-7),
    "terabyte": Config("terabyte", TERABYTE_ROWS, 64, 4096, 1,
                       records=80_000_000, t=1e-9,
                       budget_bytes=180 * 10**9),
    # L = 512 MB is slack for the 330 MB Alibaba-shaped tables: every
    # row seen in the 5 % sample is hot (the sample-bounded maximum, 16 % of
    # the records; profiles/r2/sweep_threshold.md)
    "alibaba": Config("alibaba", ALIBABA_ROWS, 16, 1024, 0, 20, 100,
                      records=10_000_000, t=1e-7, budget_bytes=512 << 20),
}


# ----------------------------------------------------------------------------
# Zipf rank sampler + Feistel scatter
# ----------------------------------------------------------------------------
_CDF_CACHE: dict = {}


def zipf_cdf(n: int, s: float, device) -> torch.Tensor:
    """Normalised CDF of Zipf(s) on ranks 1..n (fp64): cdf[i] = P(rank <= i+1).
    Always computed on the CPU (a CUDA cumsum rounds differently, which moved
    a few inverse-CDF draws at bucket edges of 10M-row tables) and copied to
    `device`, so the same counters draw the same rows on every device."""
    key = (n, s, str(device))
    c = _CDF_CACHE.get(key)
    if c is None:
        ckey = (n, s, "cpu")
        c = _CDF_CACHE.get(ckey)
        if c is None:
            r = torch.arange(1, n + 1, dtype=torch.float64)
            w = r.pow(-s)
            c = torch.cumsum(w, 0)
            c = c / c[-1]
        if len(_CDF_CACHE) > 8:
            _CDF_CACHE.clear()
        _CDF_CACHE[ckey] = c
        c = c.to(device)
        _CDF_CACHE[key] = c
    return c


def feistel(x: torch.Tensor, n: int, seed: int) -> torch.Tensor:
    """Seeded bijection on [0, n): 4-round balanced Feistel on 2h bits with
    cycle-walking.  x: int64 tensor with values in [0, n)."""
    if n <= 1:
        return x.clone()
    bits = max(2, math.ceil(math.log2(n)))
    h = (bits + 1) // 2
    mask = (1 << h) - 1
    keys = [_s64(seed * 4 + i) for i in range(4)]

    def perm(v):
        lo = v & mask
        hi = v >> h
        for k in keys:
            f = mix64(lo * _s64(GOLDEN) + k) & mask
            lo, hi = hi ^ f, lo
        return (hi << h) | lo

    y = perm(x)
    bad = y >= n
    while bool(bad.any()):
        y = torch.where(bad, perm(y), y)
        bad = y >= n
    return y


def zipf_rows(n: int, s: float, seed: int, ctr: torch.Tensor) -> torch.Tensor:
    """Row ids in [0, n) for counters ctr: rank ~ Zipf(s) by inverse CDF,
    then scattered by the table's Feistel bijection."""
    u = uniform01(seed, ctr)
    cdf = zipf_cdf(n, s, ctr.device)
    rank0 = torch.searchsorted(cdf, u).clamp_(max=n - 1)
    return feistel(rank0, n, seed ^ 0x5EED)


# ----------------------------------------------------------------------------
# Datasets
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class Dataset:
    rows: List[int]
    dim: int
    n_records: int
    idx: torch.Tensor                 # int32 [n_lookups], sample-major
    off: Optional[torch.Tensor]       # int64 [n_records*n_tables+1] or None
    fixed_pool: int                   # pooling when off is None

    @property
    def n_tables(self) -> int:
        return len(self.rows)

    @property
    def n_lookups(self) -> int:
        return int(self.idx.numel())

    def to(self, device) -> "Dataset":
        return Dataset(self.rows, self.dim, self.n_records,
                       self.idx.to(device),
                       None if self.off is None else self.off.to(device),
                       self.fixed_pool)


def make_dataset(cfg: Config, n_records: Optional[int] = None,
                 seed: int = BASE_SEED, device="cpu",
                 chunk: int = 1 << 26, record_base: int = 0) -> Dataset:
    """Synthetic Zipf-skewed categorical stream shaped like `cfg`.

    Table z draws from Zipf(cfg.zipf_s) with its own seed (seed + z), tables
    independent.  Fixed pooling: lookup q = (r*Tn + z)*P + p uses counter q.
    Variable pooling: bag b = r*Tn + z has P_b ~ U{pool_lo..pool_hi} drawn from
    seed + 777; its lookups use counters off[b]..off[b+1)-1.
    record_base: global id of local record 0 (a rank's shard of a larger
    dataset draws exactly the records the unsharded dataset would hold)."""
    R = cfg.records if n_records is None else n_records
    Tn = cfg.n_tables
    dev = torch.device(device)
    if cfg.pool > 0:
        P = cfg.pool
        idx = torch.empty(R * Tn * P, dtype=torch.int32, device=dev)
        view = idx.view(R, Tn, P)
        for z, n in enumerate(cfg.rows):
            for r0 in range(0, R, max(1, chunk // P)):
                r1 = min(R, r0 + max(1, chunk // P))
                rr = torch.arange(r0, r1, device=dev, dtype=torch.int64) + record_base
                ctr = ((rr * Tn + z) * P).unsqueeze(1) + \
                    torch.arange(P, device=dev, dtype=torch.int64)
                view[r0:r1, z, :] = zipf_rows(n, cfg.zipf_s, seed + z,
                                              ctr).to(torch.int32)
        return Dataset(list(cfg.rows), cfg.dim, R, idx, None, P)
    # variable pooling
    nb = R * Tn
    span = cfg.pool_hi - cfg.pool_lo + 1
    b = torch.arange(nb, device=dev, dtype=torch.int64) + record_base * Tn
    sizes = cfg.pool_lo + _srl(counter_hash(seed + 777, b), 11) % span
    off = torch.zeros(nb + 1, dtype=torch.int64, device=dev)
    torch.cumsum(sizes, 0, out=off[1:])
    L = int(off[-1])
    # counters of a shard continue the global stream: offset by the lookups
    # of the records before record_base (closed form unavailable -> prefix)
    q_base = 0
    if record_base:
        bp = torch.arange(record_base * Tn, device=dev, dtype=torch.int64)
        q_base = int((cfg.pool_lo + _srl(counter_hash(seed + 777, bp), 11) % span).sum())
    idx = torch.empty(L, dtype=torch.int32, device=dev)
    for q0 in range(0, L, chunk):
        q1 = min(L, q0 + chunk)
        q = torch.arange(q0, q1, device=dev, dtype=torch.int64)
        bag = torch.searchsorted(off, q, right=True) - 1
        z = bag % Tn
        q = q + q_base
        out = torch.empty(q1 - q0, dtype=torch.int64, device=dev)
        for zz, n in enumerate(cfg.rows):
            m = z == zz
            if bool(m.any()):
                out[m] = zipf_rows(n, cfg.zipf_s, seed + zz, q[m])
        idx[q0:q1] = out.to(torch.int32)
    return Dataset(list(cfg.rows), cfg.dim, R, idx, off, 0)


def make_uniform_dataset(rows: List[int], n_records: int, pool: int,
                         seed: int, device="cpu") -> Dataset:
    """Uniform (non-skewed) indices; used for L2-defeating controls and
    edge-case tests."""
    Tn = len(rows)
    dev = torch.device(device)
    q = torch.arange(n_records * Tn * pool, device=dev, dtype=torch.int64)
    z = (q // pool) % Tn
    nrow = torch.tensor(rows, dtype=torch.int64, device=dev)[z]
    h = _srl(counter_hash(seed, q), 11)
    idx = (h % nrow).to(torch.int32)
    return Dataset(list(rows), 0, n_records, idx, None, pool)


def make_weights(n_rows: int, dim: int, seed: int = BASE_SEED + 2000,
                 device="cpu", lo=-0.05, hi=0.05,
                 chunk: int = 1 << 27) -> torch.Tensor:
    """fp32 [n_rows, dim] ~ U(lo, hi) from counter g*dim + d."""
    dev = torch.device(device)
    W = torch.empty(n_rows * dim, dtype=torch.float32, device=dev)
    for c0 in range(0, n_rows * dim, chunk):
        c1 = min(n_rows * dim, c0 + chunk)
        ctr = torch.arange(c0, c1, device=dev, dtype=torch.int64)
        W[c0:c1] = (lo + (hi - lo) * uniform01(seed, ctr)).float()
    return W.view(n_rows, dim)


def make_weight_rows(rows: torch.Tensor, dim: int, seed: int = BASE_SEED + 2000,
                     lo=-0.05, hi=0.05) -> torch.Tensor:
    """Rows `rows` (int64 global row ids) of make_weights(n, dim, seed), bit
    for bit, without drawing the others (a 48 GB Terabyte-shaped table's hot
    rows on the host)."""
    rows = torch.as_tensor(rows, dtype=torch.int64)
    ctr = (rows.unsqueeze(1) * dim + torch.arange(dim, dtype=torch.int64, device=rows.device)).reshape(-1)
    return (lo + (hi - lo) * uniform01(seed, ctr)).float().view(-1, dim)


def make_dy(n_bags: int, dim: int, seed: int = BASE_SEED + 1000,
            device="cpu") -> torch.Tensor:
    """Upstream gradient dY ~ U(-1, 1), fp32 [n_bags, dim]."""
    return make_weights(n_bags, dim, seed, device, -1.0, 1.0)


# ----------------------------------------------------------------------------
# DLRM inputs (NEXT-2): dense features, labels, random-init MLP parameters
# ----------------------------------------------------------------------------
def make_dense(n_records: int, n_dense: int, seed: int = BASE_SEED + 3000,
               device="cpu", record_base: int = 0) -> torch.Tensor:
    """Dense features fp32 [n_records, n_dense] ~ U(0, 4) (the range of
    Criteo's log(1 + x) dense features), counter (record, feature)."""
    dev = torch.device(device)
    ctr = (torch.arange(n_records, device=dev, dtype=torch.int64) + record_base).unsqueeze(1) * n_dense + \
        torch.arange(n_dense, device=dev, dtype=torch.int64)
    return (4.0 * uniform01(seed, ctr.reshape(-1))).float().view(n_records, n_dense)


def make_labels(n_records: int, n_dense: int, seed: int = BASE_SEED + 4000,
                device="cpu", record_base: int = 0, dense_seed: int = BASE_SEED + 3000) -> torch.Tensor:
    """Click labels fp32 {0, 1} [n_records] with a planted, learnable rule:
    P(click) = 0.7 if dense feature 0 (of make_dense(..., dense_seed)) > 2
    else 0.1 (about 40% positives)."""
    d0 = make_dense(n_records, n_dense, seed=dense_seed, device=device, record_base=record_base)[:, 0].double()
    dev = torch.device(device)
    u = uniform01(seed, torch.arange(n_records, device=dev, dtype=torch.int64) + record_base)
    p = torch.where(d0 > 2.0, torch.full_like(d0, 0.7), torch.full_like(d0, 0.1))
    return (u < p).float()


def dlrm_dims(n_dense: int, bottom, top, n_tables: int, dim: int):
    """[(in, out)] of every bottom then top layer (flat-parameter order)."""
    dims, prev = [], n_dense
    for w in bottom:
        dims.append((prev, w))
        prev = w
    F = n_tables + 1
    prev = dim + F * (F - 1) // 2
    for w in top:
        dims.append((prev, w))
        prev = w
    return dims


def make_dlrm_params(dims, seed: int = BASE_SEED + 5000, device="cpu") -> torch.Tensor:
    """Random-init flat parameters (per layer W [out][in] then b [out]),
    U(-1/sqrt(in), 1/sqrt(in)) like PyTorch's Linear default."""
    dev = torch.device(device)
    parts, o = [], 0
    for i, n in dims:
        k = (i * n + n)
        ctr = torch.arange(o, o + k, device=dev, dtype=torch.int64)
        a = 1.0 / (i ** 0.5)
        parts.append((-a + 2 * a * uniform01(seed, ctr)).float())
        o += k
    return torch.cat(parts)


def dlrm_pad(flat: torch.Tensor, dims) -> torch.Tensor:
    """Canonical flat parameters (per layer W [out][in], b [out]) -> the
    library's layout (W rows padded to ld = in rounded up to 4 floats, pad
    entries 0; include/fae.h fae_dlrm)."""
    parts, o = [], 0
    for i, n in dims:
        ld = (i + 3) // 4 * 4
        W = flat[o:o + n * i].view(n, i)
        o += n * i
        Wp = torch.zeros(n, ld, dtype=flat.dtype, device=flat.device)
        Wp[:, :i] = W
        parts += [Wp.reshape(-1), flat[o:o + n]]
        o += n
    return torch.cat(parts)


def dlrm_unpad(flat: torch.Tensor, dims) -> torch.Tensor:
    """The library's padded layout -> canonical flat parameters."""
    parts, o = [], 0
    for i, n in dims:
        ld = (i + 3) // 4 * 4
        parts.append(flat[o:o + n * ld].view(n, ld)[:, :i].reshape(-1))
        o += n * ld
        parts.append(flat[o:o + n])
        o += n
    return torch.cat(parts)
