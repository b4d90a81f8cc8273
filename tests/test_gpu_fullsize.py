"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (FaePipeline with the bench's arguments), against the oracle.

* test_two_select_levels: 3M records force the sampler's second radix-select
  level (> 4096 candidates after the first 8-bit digit), single rank; every
  stage bit-exact.
* test_fullsize_parity: the Kaggle- (45M records, FIXED_T t = 1e-7),
  Terabyte- (80M, BUDGET_EXACT 180 GB) and Alibaba-shaped (10M, offsets,
  BUDGET_EXACT 512 MB) workloads.  Bit-exact against the oracle over the WHOLE
  dataset: sample ids, loggers, T, the threshold result (K, kmin, H, base),
  the remap of every row, hot_ids / cold_ids; the hot CSR on a seeded sample
  of hot records (oracle.pack of exactly those records); then three hot
  batches from the middle of the run trained from the extracted table vs the
  oracle's sequential SGD (1e-5 / 1e-6), the batch contents taken from the
  oracle's own classification.  The oracle runs its OpenMP build
  (bit-identical to the serial build, tests/test_oracle.py).
"""
import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu

ATOL, RTOL = 1e-6, 1e-5


def close(gpu, ref):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(gpu - ref)
    bound = ATOL + RTOL * np.abs(ref)
    return bool(np.all(err <= bound)), float((err - bound).max(initial=-1))


@pytest.fixture
def omp():
    oracle.use_omp(True)
    yield
    oracle.use_omp(False)


def _sub_csr(ds, recs):
    """CSR of the records `recs` (in that order), host numpy."""
    Tn = ds.n_tables
    idx = ds.idx.numpy() if hasattr(ds.idx, "numpy") else ds.idx
    if ds.off is None:
        P = ds.fixed_pool
        v = idx.reshape(ds.n_records, Tn * P)[recs].reshape(-1)
        return v, None, P
    off = ds.off.numpy()
    parts, sizes = [], []
    for r in recs:
        lo, hi = off[r * Tn], off[(r + 1) * Tn]
        parts.append(idx[lo:hi])
        sizes.append(np.diff(off[r * Tn:(r + 1) * Tn + 1]))
    sub_off = np.concatenate([[0], np.cumsum(np.concatenate(sizes))]).astype(np.int64)
    return np.concatenate(parts).astype(np.int32), sub_off, 0


def test_two_select_levels(omp):
    from paper_2103_00686_b200.pipeline import FaePipeline
    import paper_2103_00686_b200 as m
    dev = torch.device("cuda", 0)
    cfg = gen.CONFIGS["tiny"]
    R, x, seed, t = 3_000_000, 5.0, 99, 1e-4
    ds = gen.make_dataset(cfg, n_records=R, seed=12, device=dev)
    pipe = FaePipeline(cfg.rows, cfg.dim, cfg.batch, 1)
    samp = torch.empty(R, dtype=torch.int64, device=dev)
    counts = torch.empty(sum(cfg.rows), dtype=torch.int32, device=dev)
    T, ns = m.fae_profile(pipe.ctx, cfg.rows, cfg.dim, ds.idx, None, 1, R, x, seed, counts, samp)
    h = ds.to("cpu")
    s_ref = oracle.sample(R, x, seed)
    assert ns == len(s_ref) == 150_000
    assert np.array_equal(samp[:ns].cpu().numpy(), s_ref)
    c_ref, T_ref, _ = oracle.histogram(h.rows, h.idx, None, 1, R, s_ref)
    assert np.array_equal(counts.cpu().numpy().view(np.uint32), c_ref) and list(T) == list(T_ref)
    prep = pipe.preprocess(ds.idx, None, R, x_pct=x, seed=seed, t=t, small_table_bytes=0)
    kmin = oracle.kmin_fixed_t(h.rows, cfg.dim, 0, T_ref, t, x)
    rm, base, H = oracle.remap(h.rows, oracle.tag_rows(h.rows, cfg.dim, 0, c_ref, kmin))
    assert prep.thresh["H_total"] == H
    flag = oracle.classify(h.rows, h.idx, None, 1, R, rm)
    pk = oracle.pack(h.rows, h.idx, None, 1, R, rm, flag)
    assert prep.packed["n_hot"] == pk["n_hot"]
    assert np.array_equal(prep.hot_ids[:pk["n_hot"]].cpu().numpy(), pk["hot_ids"])
    assert np.array_equal(prep.cold_ids[:pk["n_cold"]].cpu().numpy(), pk["cold_ids"])
    assert np.array_equal(prep.hot_idx[:pk["n_hot_lookups"]].cpu().numpy(), pk["hot_idx"])


@pytest.mark.parametrize("name", ["kaggle", "terabyte", "alibaba"])
def test_fullsize_parity(omp, name):
    import paper_2103_00686_b200 as m
    from paper_2103_00686_b200.pipeline import FaePipeline
    dev = torch.device("cuda", 0)
    cfg = gen.CONFIGS[name]
    R, x, seed = cfg.records, 5.0, 1                      # bench.py's defaults
    Tn, D, B = cfg.n_tables, cfg.dim, cfg.batch
    ds = gen.make_dataset(cfg, n_records=R, device=dev)
    # --- GPU, exactly as bench.py's step ---
    pipe = FaePipeline(cfg.rows, D, B, cfg.pool, max_pool=max(cfg.pool_hi, 1), device=0)
    mode = m.BUDGET_EXACT if cfg.budget_bytes else m.FIXED_T
    samp = torch.empty(R, dtype=torch.int64, device=dev)
    counts = torch.empty(sum(cfg.rows), dtype=torch.int32, device=dev)
    T, ns = m.fae_profile(pipe.ctx, cfg.rows, D, ds.idx, ds.off, cfg.pool, R, x, seed, counts, samp)
    samp_g = samp[:ns].cpu().numpy()
    del samp
    counts_g = counts.cpu().numpy().view(np.uint32)
    prep = pipe.preprocess(ds.idx, ds.off, R, x_pct=x, seed=seed, mode=mode, t=cfg.t,
                           budget_bytes=cfg.budget_bytes, small_table_bytes=cfg.small_bytes)
    remap_g = torch.empty(sum(cfg.rows), dtype=torch.int32, device=dev)
    m.fae_threshold(pipe.ctx, cfg.rows, D, prep.counts, prep.T, x, mode=mode, t=cfg.t,
                    budget_bytes=cfg.budget_bytes, small_table_bytes=cfg.small_bytes, remap_out=remap_g)
    remap_g = remap_g.cpu().numpy()
    pk_g = prep.packed
    hot_ids_g = prep.hot_ids[:pk_g["n_hot"]].cpu().numpy()
    cold_ids_g = prep.cold_ids[:pk_g["n_cold"]].cpu().numpy()
    h = ds.to("cpu")
    # --- oracle over the whole dataset ---
    s_ref = oracle.sample(R, x, seed)
    assert ns == len(s_ref) and np.array_equal(samp_g, s_ref)
    del samp_g
    c_ref, T_ref, st = oracle.histogram(h.rows, h.idx, h.off, h.fixed_pool, R, s_ref)
    assert st == 0
    assert list(T) == list(T_ref) and list(prep.T) == list(T_ref)
    assert np.array_equal(counts_g, c_ref)
    del counts_g
    if cfg.budget_bytes:
        r = oracle.budget_exact(h.rows, D, cfg.small_bytes, c_ref, T_ref, x, cfg.budget_bytes)
        assert r["status"] == 0
        kmin = r["kmin"]
        assert prep.thresh["K"] == r["K"] and prep.thresh["t_final"] == r["t_final"]
        assert prep.thresh["budget_slack"] == r["slack"]
    else:
        kmin = oracle.kmin_fixed_t(h.rows, D, cfg.small_bytes, T_ref, cfg.t, x)
    assert [int(v) for v in prep.thresh["kmin"]] == [int(v) for v in kmin]
    rm, base, H = oracle.remap(h.rows, oracle.tag_rows(h.rows, D, cfg.small_bytes, c_ref, kmin))
    del c_ref
    assert prep.thresh["H_total"] == H and list(prep.thresh["base"]) == list(base)
    assert np.array_equal(remap_g, rm)
    del remap_g
    flag = oracle.classify(h.rows, h.idx, h.off, h.fixed_pool, R, rm)
    hot_ref = np.nonzero(flag)[0]
    assert pk_g["n_hot"] == len(hot_ref) and pk_g["n_cold"] == R - len(hot_ref)
    assert np.array_equal(hot_ids_g, hot_ref)
    assert np.array_equal(cold_ids_g, np.nonzero(flag == 0)[0])
    del cold_ids_g, flag
    # hot CSR on a seeded sample of hot records
    rng = np.random.default_rng(5)
    ks = np.sort(rng.choice(len(hot_ref), min(20_000, len(hot_ref)), replace=False))
    sub_idx, sub_off, P = _sub_csr(h, hot_ref[ks])
    pk_s = oracle.pack(h.rows, sub_idx, sub_off, P, len(ks), rm, np.ones(len(ks), np.uint8))
    hot_idx_g = prep.hot_idx
    if h.off is None:
        got = hot_idx_g.view(-1, Tn * P)[torch.from_numpy(ks).to(dev)].cpu().numpy().reshape(-1)
        assert np.array_equal(got, pk_s["hot_idx"])
    else:
        hot_off_g = prep.hot_off
        lo = hot_off_g[torch.from_numpy(ks * Tn).to(dev)].cpu().numpy()
        hi = hot_off_g[torch.from_numpy((ks + 1) * Tn).to(dev)].cpu().numpy()
        flat = hot_idx_g[:pk_g["n_hot_lookups"]].cpu().numpy()
        got = np.concatenate([flat[a:b] for a, b in zip(lo, hi)])
        assert np.array_equal(got, pk_s["hot_idx"])
        bag_sizes = np.concatenate([np.diff(hot_off_g[k * Tn:(k + 1) * Tn + 1].cpu().numpy()) for k in ks[:200]])
        ref_sizes = np.diff(pk_s["hot_off"])[:200 * Tn]
        assert np.array_equal(bag_sizes, ref_sizes)
    # --- three hot batches from the middle, training loop as in the bench ---
    nbt = pk_g["n_hot_batches"]
    first, nb = nbt // 2, 3
    hot_rows = np.nonzero(rm >= 0)[0]
    W_ref = gen.make_weight_rows(torch.from_numpy(hot_rows), D).numpy()   # == extract(W, rm)
    W = gen.make_weights(sum(cfg.rows), D, device=dev)
    W_hot = pipe.extract(W, prep)
    del W
    torch.cuda.empty_cache()
    pipe.group(prep)
    S = B * Tn
    dY = gen.make_dy(nb * S, D, seed=77).view(nb, S, D)
    Y = torch.zeros(S, D, device=dev)
    pipe.train(W_hot, first, nb, dY.to(dev), Y, 0.01)
    pipe.ctx.check()
    for i in range(nb):
        b = first + i
        recs = hot_ref[b * B: min((b + 1) * B, len(hot_ref))]
        sub_idx, sub_off, P = _sub_csr(h, recs)
        pk_b = oracle.pack(h.rows, sub_idx, sub_off, P, len(recs), rm, np.ones(len(recs), np.uint8))
        n_bags = len(recs) * Tn
        W_ref, st = oracle.emb_bwd_sgd(W_ref, pk_b["hot_idx"], pk_b["hot_off"], P, n_bags,
                                       dY[i, :n_bags].numpy(), 0.01)
        assert st == 0
    ok, worst = close(W_hot.cpu().numpy(), W_ref)
    assert ok, worst
