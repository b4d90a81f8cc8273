"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Integer stages (sample, histogram, threshold, remap, classify, pack,
extract) must be bit-exact.  fp32 stages (pooled Y, updated W_hot) must be
within |gpu - oracle| <= 1e-6 + 1e-5 * |oracle| (BASELINE.json north_star).
Inputs are the seeded generators of gen/, identical bits on both sides.
"""
import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu

ATOL, RTOL = 1e-6, 1e-5


def fae():
    import paper_2103_00686_b200 as m
    return m


def close(gpu, ref):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(gpu - ref)
    bound = ATOL + RTOL * np.abs(ref)
    return bool(np.all(err <= bound)), float((err - bound).max(initial=-1))


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def mkctx(rows, dim, batch_lookups, batch_bags, world=1):
    return fae().fae_create(0, max_tables=len(rows), max_rows=sum(rows),
                            max_batch_lookups=batch_lookups,
                            max_batch_bags=batch_bags, max_dim=max(dim, 4),
                            max_world=world)


# ----------------------------------------------------------------------------
# a8 forward / a9-a10 backward + SGD on hot batches
# ----------------------------------------------------------------------------
def _hot_batch(H, n_bags, pool, dim, seed, var=False, zipf=True):
    g = torch.Generator().manual_seed(seed)
    if var:
        sizes = torch.randint(0, 2 * pool + 1, (n_bags,), generator=g)
        off = torch.zeros(n_bags + 1, dtype=torch.int64)
        off[1:] = torch.cumsum(sizes, 0)
        L = int(off[-1])
    else:
        off = None
        L = n_bags * pool
    if zipf:
        u = gen.uniform01(seed, torch.arange(L))
        cdf = gen.zipf_cdf(H, 1.1, "cpu")
        idx = gen.feistel(torch.searchsorted(cdf, u).clamp(max=H - 1), H, seed).to(torch.int32)
    else:
        idx = torch.randint(0, H, (L,), generator=g, dtype=torch.int32)
    W = gen.make_weights(H, dim, seed=seed + 1)
    dY = gen.make_dy(n_bags, dim, seed=seed + 2)
    return W, idx, off, dY


CASES = [
    # (H, n_bags, pool, dim, var)  -- several tiles + ragged tails
    (1000, 128 * 4, 1, 16, False),          # tiny-shaped hot batch
    (50_000, 2048 * 26, 1, 16, False),      # Kaggle-shaped hot batch (S = L = 53,248)
    (200_000, 4096 * 26, 1, 64, False),     # Terabyte-shaped hot batch (L = 106,496, D = 64)
    (300_000, 1024 * 3, 60, 16, True),      # Alibaba-shaped multi-hot bags (~180k lookups)
    (777, 333, 3, 32, False),               # ragged
    (5000, 1000, 7, 128, True),             # D = 128, variable incl. empty bags
    (4096, 500, 2, 4, False),               # D = 4
]


@pytest.mark.parametrize("H,n_bags,pool,dim,var", CASES)
def test_fwd_bwd_parity(dev, H, n_bags, pool, dim, var):
    W, idx, off, dY = _hot_batch(H, n_bags, pool, dim, seed=H + n_bags, var=var)
    L = idx.numel()
    ctx = mkctx([H], dim, max(L, 1), n_bags)
    Wd, idxd, dYd = W.to(dev), idx.to(dev), dY.to(dev)
    offd = off.to(dev) if off is not None else None
    P = 0 if var else pool
    Y = torch.empty(n_bags, dim, device=dev)
    fae().fae_emb_fwd(ctx, Wd, idxd, offd, P, n_bags, Y)
    Yref, st = oracle.emb_fwd(W, idx, off, P, n_bags)
    assert st == 0
    ok, worst = close(Y.cpu().numpy(), Yref)
    assert ok, f"fwd worst excess {worst}"
    if pool == 1 and not var:
        assert torch.equal(Y.cpu(), W[idx.long()])          # single lookup: bit copy
    lr = 0.01
    fae().fae_emb_bwd_update(ctx, Wd, idxd, offd, P, n_bags, dYd, lr)
    ctx.check()
    Wref, st = oracle.emb_bwd_sgd(W, idx, off, P, n_bags, dY, lr)
    Wg = Wd.cpu().numpy()
    ok, worst = close(Wg, Wref)
    assert ok, f"bwd worst excess {worst}"
    touched = np.zeros(H, bool)
    touched[idx.numpy()] = True
    assert np.array_equal(Wg[~touched], W.numpy()[~touched])   # untouched: bit-identical


def test_bwd_deterministic(dev):
    W, idx, _, dY = _hot_batch(20_000, 2048 * 26, 1, 16, seed=5)
    ctx = mkctx([20_000], 16, idx.numel(), 2048 * 26)
    outs = []
    for _ in range(3):
        Wd = W.to(dev)
        fae().fae_emb_bwd_update(ctx, Wd, idx.to(dev), None, 1, 2048 * 26, dY.to(dev), 0.01)
        outs.append(Wd.cpu())
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


def test_step_edge_cases(dev):
    m = fae()
    ctx = mkctx([100], 16, 1000, 1000)
    W = gen.make_weights(100, 16).to(dev)
    Y = torch.empty(0, 16, device=dev)
    m.fae_emb_fwd(ctx, W, torch.empty(0, dtype=torch.int32, device=dev), None, 1, 0, Y)
    m.fae_emb_bwd_update(ctx, W, torch.empty(0, dtype=torch.int32, device=dev), None, 1, 0,
                         torch.empty(0, 16, device=dev), 0.1)
    ctx.check()
    # lr = 0 leaves W bit-identical
    W0 = W.clone()
    idx = torch.randint(0, 100, (64,), dtype=torch.int32, device=dev)
    m.fae_emb_bwd_update(ctx, W, idx, None, 1, 64, torch.ones(64, 16, device=dev), 0.0)
    ctx.check()
    assert torch.equal(W, W0)
    # out-of-range index is latched
    bad = torch.tensor([0, 5, 100], dtype=torch.int32, device=dev)
    Y = torch.empty(3, 16, device=dev)
    m.fae_emb_fwd(ctx, W, bad, None, 1, 3, Y)
    with pytest.raises(m.FaeError) as e:
        ctx.check()
    assert e.value.name == "INDEX_RANGE"
    # unsupported dim / capacity
    with pytest.raises(m.FaeError):
        m.fae_emb_fwd(ctx, torch.zeros(10, 12, device=dev), idx, None, 1, 64,
                      torch.empty(64, 12, device=dev))
    with pytest.raises(m.FaeError) as e:
        m.fae_emb_fwd(ctx, W, torch.zeros(2000, dtype=torch.int32, device=dev), None, 1, 2000,
                      torch.empty(2000, 16, device=dev))
    assert e.value.name == "CAPACITY"


# ----------------------------------------------------------------------------
# a1-a7 preprocessing
# ----------------------------------------------------------------------------
def _prep_ref(ds, x, seed, mode, t=None, budget=None, small=0, dim=16):
    samp = oracle.sample(ds.n_records, x, seed)
    counts, T, st = oracle.histogram(ds.rows, ds.idx, ds.off, ds.fixed_pool, ds.n_records, samp)
    assert st == 0
    if mode == "t":
        kmin = oracle.kmin_fixed_t(ds.rows, dim, small, T, t, x)
        extra = {}
    else:
        r = oracle.budget_exact(ds.rows, dim, small, counts, T, x, budget)
        kmin, extra = r["kmin"], r
    hot = oracle.tag_rows(ds.rows, dim, small, counts, kmin)
    rm, base, H = oracle.remap(ds.rows, hot)
    flag = oracle.classify(ds.rows, ds.idx, ds.off, ds.fixed_pool, ds.n_records, rm)
    pk = oracle.pack(ds.rows, ds.idx, ds.off, ds.fixed_pool, ds.n_records, rm, flag)
    return dict(samp=samp, counts=counts, T=T, kmin=kmin, hot=hot, remap=rm, base=base,
                H=H, flag=flag, pack=pk, extra=extra)


PREP_CASES = [
    ("tiny", 10_000, 5.0, "t", 1e-3, 0),
    ("tiny", 10_000, 5.0, "t", 1e-2, 0),
    ("tiny", 10_000, 5.0, "t", 3e-2, 0),
    ("tiny", 10_000, 100.0, "t", 3e-3, 0),
    ("tiny", 10_000, 5.0, "b", 64 * 300, 0),
    ("kaggle", 60_000, 5.0, "t", 1e-7, 1 << 20),
    ("kaggle", 60_000, 5.0, "b", 512 << 20, 1 << 20),
    ("kaggle", 60_000, 5.0, "b", 20 << 20, 1 << 20),
    ("alibaba", 3_000, 5.0, "t", 1e-5, 1 << 20),
]


@pytest.mark.parametrize("cfg,R,x,mode,arg,small", PREP_CASES)
def test_preprocess_parity(dev, cfg, R, x, mode, arg, small):
    m = fae()
    c = gen.CONFIGS[cfg]
    ds = gen.make_dataset(c, n_records=R, seed=11)
    seed = 77
    ref = _prep_ref(ds, x, seed, mode, t=arg if mode == "t" else None,
                    budget=arg if mode == "b" else None, small=small)
    ctx = mkctx(ds.rows, 16, c.batch * c.n_tables * max(c.pool, c.pool_hi, 1), c.batch * c.n_tables)
    dd = ds.to(dev)
    counts = torch.empty(sum(ds.rows), dtype=torch.int32, device=dev)
    samp = torch.empty(max(R, 1), dtype=torch.int64, device=dev)
    T, ns = m.fae_profile(ctx, ds.rows, 16, dd.idx, dd.off, ds.fixed_pool, R, x, seed, counts, samp)
    assert ns == len(ref["samp"])
    assert np.array_equal(samp[:ns].cpu().numpy(), ref["samp"])
    assert T == list(ref["T"])
    assert np.array_equal(counts.cpu().numpy().view(np.uint32), ref["counts"])
    remap = torch.empty(sum(ds.rows), dtype=torch.int32, device=dev)
    if mode == "t":
        th = m.fae_threshold(ctx, ds.rows, 16, counts, T, x, mode=m.FIXED_T, t=arg,
                             small_table_bytes=small, remap_out=remap)
    else:
        th = m.fae_threshold(ctx, ds.rows, 16, counts, T, x, mode=m.BUDGET_EXACT, budget_bytes=arg,
                             small_table_bytes=small, remap_out=remap)
        assert th["K"] == ref["extra"]["K"]
        assert th["t_final"] == ref["extra"]["t_final"]
        assert th["budget_slack"] == ref["extra"]["slack"]
    assert th["kmin"] == [int(v) for v in ref["kmin"]]
    assert th["H_total"] == ref["H"]
    assert th["base"] == [int(v) for v in ref["base"]]
    assert np.array_equal(remap.cpu().numpy(), ref["remap"])
    hot_ids = torch.empty(R, dtype=torch.int64, device=dev)
    cold_ids = torch.empty(R, dtype=torch.int64, device=dev)
    hot_idx = torch.empty(max(ds.n_lookups, 1), dtype=torch.int32, device=dev)
    hot_off = torch.empty(R * ds.n_tables + 1, dtype=torch.int64, device=dev) if ds.off is not None else None
    pk = m.fae_classify(ctx, ds.rows, 16, dd.idx, dd.off, ds.fixed_pool, R, c.batch,
                        hot_ids, cold_ids, hot_idx, hot_off)
    rp = ref["pack"]
    assert pk["n_hot"] == rp["n_hot"] and pk["n_cold"] == rp["n_cold"]
    assert pk["n_hot_lookups"] == rp["n_hot_lookups"]
    assert np.array_equal(hot_ids[:pk["n_hot"]].cpu().numpy(), rp["hot_ids"])
    assert np.array_equal(cold_ids[:pk["n_cold"]].cpu().numpy(), rp["cold_ids"])
    assert np.array_equal(hot_idx[:pk["n_hot_lookups"]].cpu().numpy(), rp["hot_idx"])
    if hot_off is not None:
        assert np.array_equal(hot_off[:pk["n_hot"] * ds.n_tables + 1].cpu().numpy(), rp["hot_off"])
    # a7 extract: bit copy
    W = gen.make_weights(sum(ds.rows), 16)
    W_hot = torch.empty(max(th["H_total"], 1), 16, device=dev)
    m.fae_extract(ctx, W.to(dev), W_hot)
    ctx.check()
    assert np.array_equal(W_hot[:th["H_total"]].cpu().numpy(), oracle.extract(W, ref["remap"], ref["H"]))


def test_estimate_parity(dev):
    m = fae()
    c = gen.CONFIGS["kaggle"]
    ds = gen.make_dataset(c, n_records=200_000, seed=3)
    x, seed = 5.0, 9
    ctx = mkctx(ds.rows, 16, 2048 * 26, 2048 * 26)
    dd = ds.to(dev)
    counts = torch.empty(sum(ds.rows), dtype=torch.int32, device=dev)
    T, ns = m.fae_profile(ctx, ds.rows, 16, dd.idx, None, 1, ds.n_records, x, seed, counts)
    th = m.fae_threshold(ctx, ds.rows, 16, counts, T, x, mode=m.FIXED_T, t=1e-7,
                         want_estimate=True, chunk_seed=1234, t_quantile=3.6007)
    cnt = counts.cpu().numpy().view(np.uint32)
    base = np.concatenate([[0], np.cumsum(ds.rows)])
    for z, n in enumerate(ds.rows):
        if th["is_small"][z]:
            continue
        e = oracle.estimate(cnt[base[z]:base[z + 1]], th["kmin"][z], 35, 1024, 1234 ^ z, 3.6007)
        assert th["est_mean"][z] == e["ybar"]
        assert th["est_sd"][z] == e["s"]
        assert th["est_lo"][z] == e["lo"] and th["est_hi"][z] == e["hi"]
        assert th["est_rows"][z] == e["est"]
        assert bool(th["est_exact"][z]) == e["exact"]


def test_preprocess_errors(dev):
    m = fae()
    ds = gen.make_dataset(gen.CONFIGS["tiny"], n_records=100)
    dd = ds.to(dev)
    ctx = mkctx(ds.rows, 16, 1000, 1000)
    counts = torch.empty(sum(ds.rows), dtype=torch.int32, device=dev)
    for bad_x in (0.0, -1.0, 100.5):
        with pytest.raises(m.FaeError) as e:
            m.fae_profile(ctx, ds.rows, 16, dd.idx, None, 1, 100, bad_x, 1, counts)
        assert e.value.name == "INVALID_ARG"
    T, _ = m.fae_profile(ctx, ds.rows, 16, dd.idx, None, 1, 100, 100.0, 1, counts)
    with pytest.raises(m.FaeError) as e:
        m.fae_threshold(ctx, ds.rows, 16, counts, T, 5.0, mode=m.FIXED_T, t=0.0)
    assert e.value.name == "INVALID_ARG"
    with pytest.raises(m.FaeError) as e:
        m.fae_threshold(ctx, ds.rows, 16, counts, T, 5.0, mode=m.BUDGET_EXACT, budget_bytes=10,
                        small_table_bytes=1 << 20)
    assert e.value.name == "BUDGET_INFEASIBLE"
    bad = dd.idx.clone()
    bad[7] = 5000
    with pytest.raises(m.FaeError) as e:
        m.fae_profile(ctx, ds.rows, 16, bad, None, 1, 100, 100.0, 1, counts)
    assert e.value.name == "INDEX_RANGE"
    with pytest.raises(m.FaeError) as e:
        m.fae_classify(ctx, ds.rows, 16, dd.idx, None, 1, 100, 0,
                       torch.empty(100, dtype=torch.int64, device=dev),
                       torch.empty(100, dtype=torch.int64, device=dev),
                       torch.empty(400, dtype=torch.int32, device=dev))
    assert e.value.name == "INVALID_ARG"


def test_sync_identity_world1(dev):
    """fae_sync_hot_grads over a 1-rank NCCL comm runs the gather + merge path
    and must return the input list unchanged (sorted, unique)."""
    m = fae()
    ctx = mkctx([1000], 16, 4096, 4096, world=1)
    m.fae_comm_init(ctx, m.fae_get_nccl_id(), 0, 1)
    rows = torch.tensor(sorted(np.random.default_rng(0).choice(1000, 300, replace=False)),
                        dtype=torch.int32, device=dev)
    vals = gen.make_dy(300, 16).to(dev)
    r0, v0 = rows.clone(), vals.clone()
    cap_rows = torch.zeros(4096, dtype=torch.int32, device=dev)
    cap_vals = torch.zeros(4096, 16, device=dev)
    cap_rows[:300] = rows
    cap_vals[:300] = vals
    n = m.fae_sync_hot_grads(ctx, cap_rows, cap_vals, 300)
    assert n == 300
    assert torch.equal(cap_rows[:300], r0) and torch.equal(cap_vals[:300], v0)


def test_pipeline_end_to_end_kaggle(dev):
    """Kaggle-shaped: full a1-a10 over 100k records, first 3 hot batches
    trained; W_hot after 3 sequential SGD steps vs the oracle."""
    from paper_2103_00686_b200.pipeline import FaePipeline
    c = gen.CONFIGS["kaggle"]
    R = 100_000
    ds = gen.make_dataset(c, n_records=R, seed=21)
    dd = ds.to(dev)
    pipe = FaePipeline(ds.rows, 16, c.batch, 1)
    prep = pipe.preprocess(dd.idx, None, R, x_pct=5.0, seed=3, t=1e-6)
    W = gen.make_weights(sum(ds.rows), 16)
    W_hot = pipe.extract(W.to(dev), prep)
    ref = _prep_ref(ds, 5.0, 3, "t", t=1e-6, small=1 << 20)
    Wref = oracle.extract(W, ref["remap"], ref["H"])
    lr = 0.05
    Y = torch.empty(c.batch * 26, 16, device=dev)
    hot_idx = ref["pack"]["hot_idx"]
    for i in range(min(3, prep.packed["n_hot_batches"])):
        idx, off, n_bags = pipe.batch_args(prep, i)
        dY = gen.make_dy(n_bags, 16, seed=100 + i)
        pipe.step(W_hot, prep, i, Y[:n_bags], dY.to(dev), lr)
        bi = hot_idx[i * c.batch * 26:(i * c.batch * 26) + n_bags]
        Yref, _ = oracle.emb_fwd(Wref, bi, None, 1, n_bags)
        ok, worst = close(Y[:n_bags].cpu().numpy(), Yref)
        assert ok, worst
        Wref, _ = oracle.emb_bwd_sgd(Wref, bi, None, 1, n_bags, dY, lr)
    pipe.ctx.check()
    ok, worst = close(W_hot.cpu().numpy(), Wref)
    assert ok, worst


# Terabyte-shaped (26 tables with the same skew of sizes, D = 64), scaled down
TB_SMALL = gen.Config("tb-small", [max(3, r // 200) for r in gen.TERABYTE_ROWS], 64, 512, 1,
                      records=30_000, t=1e-6)


@pytest.mark.parametrize("where", ["end", "mid"])
@pytest.mark.parametrize("mode", ["graph", "fused", "persist"])
@pytest.mark.parametrize("cfg,R,t,small", [("kaggle", 100_000, 1e-6, 1 << 20),
                                           ("alibaba", 20_000, 1e-5, 1 << 20),
                                           ("tiny", 10_000, 1e-2, 0),
                                           ("tb-small", 30_000, 1e-6, 1 << 20)])
def test_grouped_training(dev, cfg, R, t, small, mode, where, monkeypatch):
    """fae_group_batches + fae_train_hot_batches (graph replay with a device
    cursor, the fused graph step, or the persistent grid-barrier kernel) ==
    the standalone per-step calls bit for bit, and == the oracle's
    sequential SGD within tolerance; includes the ragged last batch."""
    from paper_2103_00686_b200.pipeline import FaePipeline
    # read at fae_create
    monkeypatch.setenv("FAE_FUSED", "1" if mode == "fused" else "0")
    monkeypatch.setenv("FAE_PERSIST", "1" if mode == "persist" else "0")
    c = TB_SMALL if cfg == "tb-small" else gen.CONFIGS[cfg]
    ds = gen.make_dataset(c, n_records=R, seed=5)
    dd = ds.to(dev)
    pipe = FaePipeline(ds.rows, c.dim, c.batch, c.pool, max_pool=max(c.pool_hi, 1))
    prep = pipe.preprocess(dd.idx, dd.off, R, x_pct=5.0, seed=2, t=t, small_table_bytes=small)
    W = gen.make_weights(sum(ds.rows), c.dim)
    W_hot = pipe.extract(W.to(dev), prep).clone()
    W_std = W_hot.clone()
    nbt = prep.packed["n_hot_batches"]
    nb = min(24 if mode == "persist" else 5, nbt)
    # a run ending at the grouping's last batch, or one in the middle (its
    # last step must not follow the segment links into the batch after it)
    first = nbt - nb if where == "end" else (nbt - nb) // 2
    S = c.batch * c.n_tables
    dY = gen.make_dy(nb * S, c.dim, seed=9).view(nb, S, c.dim).to(dev)
    lr = 0.05
    pipe.group(prep)
    from paper_2103_00686_b200 import fae_group_info
    want = {"graph": 0, "fused": 1, "persist": 2}[mode] if c.pool == 1 else 0
    assert fae_group_info(pipe.ctx)["fused"] == want
    Y = torch.zeros(S, c.dim, device=dev)
    pipe.train(W_hot, first, nb, dY, Y, lr)
    pipe.ctx.check()
    Y2 = torch.zeros(S, c.dim, device=dev)
    for i in range(nb):
        _, _, n_bags = pipe.batch_args(prep, first + i)
        pipe.step(W_std, prep, first + i, Y2[:n_bags], dY[i, :n_bags], lr)
    pipe.ctx.check()
    assert torch.equal(W_hot, W_std)
    assert torch.equal(Y, Y2)
    # oracle: sequential SGD over the same batches
    ref = _prep_ref(ds, 5.0, 2, "t", t=t, small=small, dim=c.dim)
    Wr = oracle.extract(W, ref["remap"], ref["H"])
    pk = ref["pack"]
    Tn = c.n_tables
    for i in range(nb):
        b = first + i
        r0, r1 = b * c.batch, min((b + 1) * c.batch, pk["n_hot"])
        n_bags = (r1 - r0) * Tn
        if ds.off is None:
            bi, off, P = pk["hot_idx"][r0 * Tn * c.pool: r1 * Tn * c.pool], None, c.pool
        else:
            bi, off, P = pk["hot_idx"], pk["hot_off"][r0 * Tn: r1 * Tn + 1], 0
        Wr, _ = oracle.emb_bwd_sgd(Wr, bi, off, P, n_bags, dY[i, :n_bags].cpu(), lr)
    ok, worst = close(W_hot.cpu().numpy(), Wr)
    assert ok, worst


@pytest.mark.parametrize("budget", [4 << 20, 8 << 20, 1 << 40])
def test_clt_search_parity(dev, budget):
    """NEXT-4: the CLT-driven statistical optimizer (R27) on the
    device == oracle.clt_search bit for bit (t_final, cutoffs, hot rows,
    remap), on the device's own loggers; includes the slack case (1 TB)."""
    m = fae()
    c = gen.CONFIGS["kaggle"]
    ds = gen.make_dataset(c, n_records=400_000, seed=4)
    x, seed = 5.0, 3
    ctx = mkctx(ds.rows, 16, 2048 * 26, 2048 * 26)
    dd = ds.to(dev)
    counts = torch.empty(sum(ds.rows), dtype=torch.int32, device=dev)
    T, _ = m.fae_profile(ctx, ds.rows, 16, dd.idx, None, 1, ds.n_records, x, seed, counts)
    remap = torch.empty(sum(ds.rows), dtype=torch.int32, device=dev)
    th = m.fae_threshold(ctx, ds.rows, 16, counts, T, x, mode=m.CLT_SEARCH, budget_bytes=budget,
                         chunk_seed=77, t_quantile=3.6007, remap_out=remap)
    cnt = counts.cpu().numpy().view(np.uint32)
    r = oracle.clt_search(ds.rows, 16, 1 << 20, cnt, T, x, budget, chunk_seed=77, t_q=3.6007)
    assert r["status"] == 0
    assert th["t_final"] == r["t_final"]
    assert th["budget_slack"] == r["slack"]
    assert [int(k) for k in th["kmin"]] == [int(k) for k in r["kmin"]]
    hot = oracle.tag_rows(ds.rows, 16, 1 << 20, cnt, r["kmin"])
    rm, base, H = oracle.remap(ds.rows, hot)
    assert th["H_total"] == H and list(th["base"]) == list(base)
    assert np.array_equal(remap.cpu().numpy(), rm)


def test_clt_search_infeasible_gpu(dev):
    m = fae()
    rows = [40 * 1024]
    ctx = mkctx(rows, 16, 1024, 1024)
    counts = torch.full((rows[0],), 1000, dtype=torch.int32, device=dev)
    with pytest.raises(m.FaeError) as e:
        m.fae_threshold(ctx, rows, 16, counts, [100], 5.0, mode=m.CLT_SEARCH, budget_bytes=1000)
    assert e.value.name == "BUDGET_INFEASIBLE"


@pytest.mark.parametrize("cfg,R,pool", [("kaggle", 60_000, 1), ("tb-small", 30_000, 1), ("tiny", 10_000, 3)])
def test_grouping_unit_path_equals_generic(dev, cfg, R, pool, monkeypatch):
    """The fixed-pooling per-(batch, table) shared-memory grouping and the
    generic segmented radix passes give the same grouping: identical
    segment statistics and bit-identical training results."""
    from paper_2103_00686_b200 import fae_group_info
    from paper_2103_00686_b200.pipeline import FaePipeline
    c = TB_SMALL if cfg == "tb-small" else gen.CONFIGS[cfg]
    if pool != c.pool:
        c = gen.Config(c.name + "-p", c.rows, c.dim, c.batch, pool, records=R, t=c.t)
    ds = gen.make_dataset(c, n_records=R, seed=6)
    dd = ds.to(dev)
    W = gen.make_weights(sum(ds.rows), c.dim)
    outs = []
    for generic in ("1", "0"):
        monkeypatch.setenv("FAE_GS_GENERIC", generic)   # read at fae_create
        pipe = FaePipeline(ds.rows, c.dim, c.batch, c.pool, max_pool=max(c.pool, 1))
        prep = pipe.preprocess(dd.idx, dd.off, R, x_pct=5.0, seed=2, t=1e-6, small_table_bytes=1 << 20)
        W_hot = pipe.extract(W.to(dev), prep).clone()
        pipe.group(prep)
        info = fae_group_info(pipe.ctx)
        nb = prep.packed["n_hot_batches"]
        S = c.batch * c.n_tables
        dY = gen.make_dy(nb * S, c.dim, seed=9).view(nb, S, c.dim).to(dev)
        Y = torch.zeros(S, c.dim, device=dev)
        pipe.train(W_hot, 0, nb, dY, Y, 0.05)
        pipe.ctx.check()
        outs.append((info, W_hot.cpu(), Y.cpu()))
    assert outs[0][0] == outs[1][0]
    assert torch.equal(outs[0][1], outs[1][1]) and torch.equal(outs[0][2], outs[1][2])


@pytest.mark.parametrize("cfg", ["kaggle", "tb-small"])
def test_train_exchange_loop_world1(dev, cfg, monkeypatch):
    """The multi-rank training loop (per-step sparse-gradient exchange over
    NCCL: reduce-emit into the rank's slot, in-place all-gather, rank-ordered
    merge, replayed from a captured graph of 128 steps) on a 1-rank
    communicator == the single-GPU loop, bit for bit: more than one graph
    replay, a call split in two ranges, both merge variants (binary search /
    row-position table)."""
    m = fae()
    from paper_2103_00686_b200.pipeline import FaePipeline
    c = TB_SMALL if cfg == "tb-small" else gen.CONFIGS[cfg]
    R = 30_000 if cfg == "tb-small" else 100_000
    if cfg == "kaggle":
        c = gen.Config("kaggle-b32", c.rows, c.dim, 32, 1, records=R, t=c.t)
    ds = gen.make_dataset(c, n_records=R, seed=8)
    dd = ds.to(dev)
    W = gen.make_weights(sum(ds.rows), c.dim)
    outs = []
    for force, table in (("0", "0"), ("1", "0"), ("1", "1")):
        monkeypatch.setenv("FAE_FORCE_MERGE", force)   # read at fae_create
        monkeypatch.setenv("FAE_MERGE_TABLE", table)
        pipe = FaePipeline(ds.rows, c.dim, c.batch, c.pool, max_pool=max(c.pool, 1))
        if force == "1":
            m.fae_comm_init(pipe.ctx, m.fae_get_nccl_id(), 0, 1)
        prep = pipe.preprocess(dd.idx, dd.off, R, x_pct=5.0, seed=2, t=1e-6, small_table_bytes=1 << 20)
        W_hot = pipe.extract(W.to(dev), prep).clone()
        pipe.group(prep)
        nb = min(prep.packed["n_hot_batches"], 300)
        if cfg == "kaggle":
            assert nb > 128, "more than one replay of the captured exchange graph"
        S = c.batch * c.n_tables
        dY = gen.make_dy(nb * S, c.dim, seed=10).view(nb, S, c.dim).to(dev)
        Y = torch.zeros(S, c.dim, device=dev)
        m.fae_set_kernel_timing(pipe.ctx, 1)
        h = nb // 3
        pipe.train(W_hot, 0, h, dY[:max(h, 1)], Y, 0.05)
        pipe.train(W_hot, h, nb - h, dY[h:], Y, 0.05)
        pipe.ctx.check()
        if force == "1":
            xt = m.fae_get_exchange_timing(pipe.ctx)
            assert xt["steps"] == nb and xt["steps_timed"] == nb and xt["xcap"] > 0
            assert xt["allgather_ms"] >= 0 and xt["merge_ms"] > 0
        m.fae_set_kernel_timing(pipe.ctx, 0)
        outs.append((W_hot.cpu(), Y.cpu()))
    for o in outs[1:]:
        assert torch.equal(outs[0][0], o[0])
        assert torch.equal(outs[0][1], o[1])


def test_merge_apply_equals_sort_merge(dev, monkeypatch):
    """The rank-ordered merge kernel and the sort-based merge of the exchanged
    gradients apply the same update to W (fae_train_hot_batches through the
    exchange loop on a 1-rank communicator)."""
    m = fae()
    from paper_2103_00686_b200.pipeline import FaePipeline
    c = gen.CONFIGS["kaggle"]
    ds = gen.make_dataset(c, n_records=100_000, seed=12)
    dd = ds.to(dev)
    W = gen.make_weights(sum(ds.rows), c.dim)
    outs = []
    monkeypatch.setenv("FAE_FORCE_MERGE", "1")
    for sort in ("1", "0"):
        monkeypatch.setenv("FAE_MERGE_SORT", sort)
        pipe = FaePipeline(ds.rows, c.dim, c.batch, c.pool)
        m.fae_comm_init(pipe.ctx, m.fae_get_nccl_id(), 0, 1)
        prep = pipe.preprocess(dd.idx, None, 100_000, x_pct=5.0, seed=2, t=1e-6)
        W_hot = pipe.extract(W.to(dev), prep).clone()
        pipe.group(prep)
        nb = min(prep.packed["n_hot_batches"], 8)
        S = c.batch * c.n_tables
        dY = gen.make_dy(nb * S, c.dim, seed=11).view(nb, S, c.dim).to(dev)
        Y = torch.zeros(S, c.dim, device=dev)
        pipe.train(W_hot, 0, nb, dY, Y, 0.05)
        pipe.ctx.check()
        outs.append(W_hot.cpu())
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("host", [False, True])
def test_scatter_hot_swap_sync(dev, host):
    """NEXT-1 swap sync: after training the hot table on
    the GPU, fae_scatter_hot writes its rows back into the master tables
    (device or pinned host memory) == oracle.scatter_hot, bit for bit; cold
    rows untouched."""
    m = fae()
    from paper_2103_00686_b200.pipeline import FaePipeline
    c = gen.CONFIGS["kaggle"]
    ds = gen.make_dataset(c, n_records=100_000, seed=14)
    dd = ds.to(dev)
    pipe = FaePipeline(ds.rows, c.dim, c.batch, c.pool)
    remap = torch.empty(sum(ds.rows), dtype=torch.int32, device=dev)
    prep = pipe.preprocess(dd.idx, None, 100_000, x_pct=5.0, seed=2, t=1e-6)
    W = gen.make_weights(sum(ds.rows), c.dim)
    W_hot = pipe.extract(W.to(dev), prep).clone()
    pipe.group(prep)
    nb = min(prep.packed["n_hot_batches"], 4)
    S = c.batch * c.n_tables
    dY = gen.make_dy(nb * S, c.dim, seed=15).view(nb, S, c.dim).to(dev)
    Y = torch.zeros(S, c.dim, device=dev)
    pipe.train(W_hot, 0, nb, dY, Y, 0.05)
    # the remap of the ctx's hot set (same threshold call again, remap out)
    m.fae_threshold(pipe.ctx, ds.rows, c.dim, prep.counts, prep.T, 5.0, mode=m.FIXED_T, t=1e-6,
                    remap_out=remap)
    Wm = W.clone().pin_memory() if host else W.to(dev)
    m.fae_scatter_hot(pipe.ctx, W_hot, Wm)
    torch.cuda.synchronize()
    pipe.ctx.check()
    ref = oracle.scatter_hot(W, W_hot.cpu(), remap.cpu())
    assert np.array_equal(Wm.cpu().numpy(), ref)


ALI_SMALL = gen.Config("ali-small", gen.ALIBABA_ROWS, 16, 128, 0, 20, 100, records=20_000, t=1e-7)


@pytest.mark.parametrize("cfgname,R,t,small", [("tiny", 10_000, 1e-2, 0), ("ali-small", 20_000, 1e-7, 1 << 20)])
def test_mixed_hot_cold_schedule(dev, cfgname, R, t, small):
    """NEXT-1 end to end: hot batches on the replicated hot table, swap sync
    (fae_scatter_hot), cold batches on the full tables through the cold CSR in
    global row ids (fae_pack_cold + the standalone step calls; fixed pooling
    and explicit offsets), re-extract, more hot batches == the oracle's
    sequential SGD over the same schedule (the swaps;
    1e-5 / 1e-6)."""
    m = fae()
    from paper_2103_00686_b200.pipeline import FaePipeline
    c = ALI_SMALL if cfgname == "ali-small" else gen.CONFIGS[cfgname]
    x, seed = 5.0, 7
    ds = gen.make_dataset(c, n_records=R, seed=3)
    dd = ds.to(dev)
    Tn, D, B = c.n_tables, c.dim, c.batch
    pipe = FaePipeline(ds.rows, D, B, c.pool, max_pool=max(c.pool_hi, 1))
    prep = pipe.preprocess(dd.idx, dd.off, R, x_pct=x, seed=seed, t=t, small_table_bytes=small)
    W0 = gen.make_weights(sum(ds.rows), D)
    Wd = W0.to(dev).clone()
    W_hot = pipe.extract(Wd, prep).clone()
    n_cold = prep.packed["n_cold"]
    assert n_cold > B, "the schedule trains two cold batches"
    assert prep.packed["n_hot_batches"] >= 3, "the schedule trains three hot batches"
    cold_idx = torch.empty(max(ds.n_lookups, 1), dtype=torch.int32, device=dev)
    cold_off = torch.empty(n_cold * Tn + 1, dtype=torch.int64, device=dev) if ds.off is not None else None
    m.fae_pack_cold(pipe.ctx, ds.rows, D, dd.idx, ds.fixed_pool, R, prep.cold_ids, n_cold, cold_idx,
                    off=dd.off, cold_off=cold_off)
    # oracle side: the cold CSR by its definition (base_z + local id, bag order)
    ref = _prep_ref(ds, x, seed, "t", t=t, small=small, dim=D)
    pk, rm, H = ref["pack"], ref["remap"], ref["H"]
    assert prep.packed["n_cold"] == pk["n_cold"]
    base = np.concatenate([[0], np.cumsum(ds.rows)])
    idx_np = ds.idx.numpy()
    if ds.off is None:
        cold_ref = (idx_np.reshape(R, Tn)[pk["cold_ids"]] + base[:Tn]).reshape(-1).astype(np.int32)
        cold_off_ref = None
    else:
        off_np = ds.off.numpy()
        parts, sizes = [], []
        for r in pk["cold_ids"]:
            for z in range(Tn):
                lo, hi = off_np[r * Tn + z], off_np[r * Tn + z + 1]
                parts.append(idx_np[lo:hi] + base[z])
                sizes.append(hi - lo)
        cold_ref = np.concatenate(parts).astype(np.int32)
        cold_off_ref = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        assert np.array_equal(cold_off.cpu().numpy(), cold_off_ref)
    assert np.array_equal(cold_idx[:len(cold_ref)].cpu().numpy(), cold_ref)
    Wr_full = W0.numpy().copy()
    Wr_hot = oracle.extract(Wr_full, rm, H)
    lr = 0.05
    sched = [("hot", 0), ("hot", 1), ("cold", 0), ("cold", 1), ("hot", 2)]
    Y = torch.empty(B * Tn, D, device=dev)
    k = 0
    prev = "hot"
    for kind, i in sched:
        dY = gen.make_dy(B * Tn, D, seed=200 + k)
        k += 1
        if kind != prev:   # swap
            if kind == "cold":
                m.fae_scatter_hot(pipe.ctx, W_hot, Wd)
                Wr_full = oracle.scatter_hot(Wr_full, Wr_hot, rm)
            else:
                W_hot.copy_(pipe.extract(Wd, prep))   # refresh the replica from the master
                Wr_hot = oracle.extract(Wr_full, rm, H)
            prev = kind
        if kind == "hot":
            idx, off, nb_ = pipe.batch_args(prep, i)
            pipe.step(W_hot, prep, i, Y[:nb_], dY[:nb_].to(dev), lr)
            r0, r1 = i * B, min((i + 1) * B, pk["n_hot"])
            if ds.off is None:
                bi, boff, P = pk["hot_idx"][r0 * Tn: r1 * Tn], None, 1
            else:
                bi, boff, P = pk["hot_idx"], pk["hot_off"][r0 * Tn: r1 * Tn + 1], 0
            Wr_hot, _ = oracle.emb_bwd_sgd(Wr_hot, bi, boff, P, nb_, dY[:nb_], lr)
        else:
            r0, r1 = i * B, min((i + 1) * B, n_cold)
            nb_ = (r1 - r0) * Tn
            if ds.off is None:
                ci, coff, P = cold_idx[r0 * Tn: r1 * Tn], None, 1
                bi, boff = cold_ref[r0 * Tn: r1 * Tn], None
            else:
                ci, coff, P = cold_idx, cold_off[r0 * Tn: r1 * Tn + 1], 0
                bi, boff = cold_ref, cold_off_ref[r0 * Tn: r1 * Tn + 1]
            m.fae_emb_fwd(pipe.ctx, Wd, ci, coff, P, nb_, Y[:nb_])
            m.fae_emb_bwd_update(pipe.ctx, Wd, ci, coff, P, nb_, dY[:nb_].to(dev), lr)
            Wr_full, _ = oracle.emb_bwd_sgd(Wr_full, bi, boff, P, nb_, dY[:nb_], lr)
    m.fae_scatter_hot(pipe.ctx, W_hot, Wd)
    Wr_full = oracle.scatter_hot(Wr_full, Wr_hot, rm)
    pipe.ctx.check()
    ok, worst = close(Wd.cpu().numpy(), Wr_full)
    assert ok, worst


@pytest.mark.parametrize("cfgname,R,t,small,cap", [("tiny", 10_000, 1e-2, 0, None),
                                                  ("ali-small", 20_000, 1e-7, 1 << 20, 3)])
def test_mixed_epoch_grouped(dev, cfgname, R, t, small, cap):
    """NEXT-1 with both kinds on the graph-replayed loop (pipeline.MixedEpoch):
    cold batches grouped once in global row ids and trained on the master
    tables, hot batches on the replica, the hot rows synchronised at every
    change of kind; cold-first phases ("always begins with
    training on cold inputs") == the oracle's sequential SGD over the same
    phase order (1e-5 / 1e-6), swaps counted."""
    from paper_2103_00686_b200.pipeline import FaePipeline, MixedEpoch
    c = ALI_SMALL if cfgname == "ali-small" else gen.CONFIGS[cfgname]
    # lr of the workloads: the tolerance derivation of §8(c)
    # (fp32 sums of Zipf-head segments) assumes it; the cold side here trains
    # every cold batch, whose head rows carry thousands of lookups
    x, seed, lr = 5.0, 7, 0.01
    ds = gen.make_dataset(c, n_records=R, seed=3)
    dd = ds.to(dev)
    Tn, D, B = c.n_tables, c.dim, c.batch
    pipe = FaePipeline(ds.rows, D, B, c.pool, max_pool=max(c.pool_hi, 1))
    prep = pipe.preprocess(dd.idx, dd.off, R, x_pct=x, seed=seed, t=t, small_table_bytes=small)
    W0 = gen.make_weights(sum(ds.rows), D)
    Wd = W0.to(dev).clone()
    W_hot = pipe.extract(Wd, prep).clone()
    ep = MixedEpoch(pipe, prep, Wd, dd.idx, dd.off, R, W_hot)
    nh, nc = ep.n_hot_batches, ep.n_cold_batches
    assert nh >= 2 and nc >= 2
    ref = _prep_ref(ds, x, seed, "t", t=t, small=small, dim=D)
    pk, rm, H = ref["pack"], ref["remap"], ref["H"]
    base = np.concatenate([[0], np.cumsum(ds.rows)])
    idx_np = ds.idx.numpy()
    off_np = ds.off.numpy() if ds.off is not None else None

    def cold_batch(i):            # global-id CSR of cold batch i, by definition
        r0, r1 = i * B, min((i + 1) * B, pk["n_cold"])
        parts, sizes = [], []
        for r in pk["cold_ids"][r0:r1]:
            for z in range(Tn):
                if off_np is None:
                    v = idx_np[r * Tn + z: r * Tn + z + 1]
                else:
                    v = idx_np[off_np[r * Tn + z]: off_np[r * Tn + z + 1]]
                parts.append(v + base[z])
                sizes.append(len(v))
        bi = np.concatenate(parts).astype(np.int32)
        return bi, np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64), (r1 - r0) * Tn

    def hot_batch(i):
        r0, r1 = i * B, min((i + 1) * B, pk["n_hot"])
        if ds.off is None:
            return pk["hot_idx"][r0 * Tn: r1 * Tn], None, (r1 - r0) * Tn
        ho = pk["hot_off"][r0 * Tn: r1 * Tn + 1]
        return pk["hot_idx"][ho[0]:ho[-1]], ho - ho[0], (r1 - r0) * Tn

    h1, c1 = nh // 2, nc // 2
    phases = [("cold", 0, c1), ("hot", 0, h1), ("cold", c1, nc - c1), ("hot", h1, nh - h1)]
    if cap:   # multi-hot: a few batches per phase (fp32 sums of Zipf-head segments
        #       of thousands of lookups over a whole epoch would drift past the
        #       per-step tolerance of north_star)
        phases = [(k, f, min(n, cap)) for k, f, n in phases]
    S = B * Tn
    Y = torch.zeros(S, D, device=dev)
    Wr_full = W0.numpy().astype(np.float32).copy()
    Wr_hot = oracle.extract(Wr_full, rm, H)
    cur = "hot"
    for k, (kind, first, n) in enumerate(phases):
        dY = gen.make_dy(n * S, D, seed=500 + k).view(n, S, D)
        ep.train(kind, first, n, dY.to(dev), Y, lr)
        if kind != cur:
            if kind == "cold":
                Wr_full = oracle.scatter_hot(Wr_full, Wr_hot, rm)
            else:
                Wr_hot = oracle.extract(Wr_full, rm, H)
            cur = kind
        for j in range(n):
            if kind == "hot":
                bi, bo, nb_ = hot_batch(first + j)
                Wr_hot, st = oracle.emb_bwd_sgd(Wr_hot, bi, bo, 0 if bo is not None else 1, nb_,
                                                dY[j, :nb_].numpy(), lr)
            else:
                bi, bo, nb_ = cold_batch(first + j)
                Wr_full, st = oracle.emb_bwd_sgd(Wr_full, bi, bo, 0, nb_, dY[j, :nb_].numpy(), lr)
            assert st == 0
    ep.finish()
    Wr_full = oracle.scatter_hot(Wr_full, Wr_hot, rm)
    pipe.ctx.check()
    ep.cold.ctx.check()
    assert ep.swaps == 5    # (replica current) -> cold -> hot -> cold -> hot, then finish -> cold
    ok, worst = close(Wd.cpu().numpy(), Wr_full)
    assert ok, worst


def test_bwd_oversized_offsets_batch_latches_capacity(dev):
    """a multi-hot batch with more lookups than max_batch_lookups
    must not write past the workspace: CAPACITY is latched and W untouched."""
    m = fae()
    ctx = mkctx([1000], 16, 256, 64)
    W = gen.make_weights(1000, 16).to(dev)
    W0 = W.clone()
    off = torch.arange(0, 65 * 10, 10, dtype=torch.int64, device=dev)    # 64 bags x 10 = 640 > 256
    idx = torch.randint(0, 1000, (640,), dtype=torch.int32, device=dev)
    m.fae_emb_bwd_update(ctx, W, idx, off, 0, 64, torch.ones(64, 16, device=dev), 0.1)
    with pytest.raises(m.FaeError) as e:
        ctx.check()
    assert e.value.name == "CAPACITY"
    assert torch.equal(W, W0)


# Two-kernel step at other row widths and a batch whose forward needs several
# bag tiles per CTA: medium segments packed 4 per CTA (D = 32, 8-lane groups),
# one per CTA (D = 128), and the staged-id forward past its 1024-bag tile
# (B * Tn > 2 * SMs * 1024 bags).  All tables are small (all hot), so every
# record is a hot record and the Zipf heads give segments in every tier.
@pytest.mark.parametrize("name,dim,batch,R", [("d32", 32, 512, 6_000), ("d128", 128, 256, 3_000),
                                              ("d64-big", 64, 12_288, 26_000)])
def test_grouped_two_kernel_dims(dev, name, dim, batch, R, monkeypatch):
    """fae_train_hot_batches (graph, two-kernel step) == the standalone calls
    bit for bit and == the oracle's sequential SGD within tolerance."""
    from paper_2103_00686_b200 import fae_group_info
    from paper_2103_00686_b200.pipeline import FaePipeline
    monkeypatch.setenv("FAE_FUSED", "0")
    monkeypatch.setenv("FAE_PERSIST", "0")
    rows = [max(3, r // 20_000) for r in gen.TERABYTE_ROWS]
    c = gen.Config(name, rows, dim, batch, 1, records=R, t=1e-6)
    small = 1 << 40                                  # every table all-hot (P:L386-387 rule)
    ds = gen.make_dataset(c, n_records=R, seed=11)
    dd = ds.to(dev)
    pipe = FaePipeline(ds.rows, c.dim, c.batch, 1)
    prep = pipe.preprocess(dd.idx, None, R, x_pct=5.0, seed=3, t=c.t, small_table_bytes=small)
    assert prep.packed["n_hot"] == R
    W = gen.make_weights(sum(ds.rows), c.dim)
    W_hot = pipe.extract(W.to(dev), prep).clone()
    W_std = W_hot.clone()
    nbt = prep.packed["n_hot_batches"]
    nb = min(3, nbt)
    first = nbt - nb                                   # includes the ragged last batch
    S = c.batch * c.n_tables
    dY = gen.make_dy(nb * S, c.dim, seed=13).view(nb, S, c.dim).to(dev)
    lr = 0.05
    pipe.group(prep)
    assert fae_group_info(pipe.ctx)["fused"] == 0
    Y = torch.zeros(S, c.dim, device=dev)
    pipe.train(W_hot, first, nb, dY, Y, lr)
    pipe.ctx.check()
    Y2 = torch.zeros(S, c.dim, device=dev)
    for i in range(nb):
        _, _, n_bags = pipe.batch_args(prep, first + i)
        pipe.step(W_std, prep, first + i, Y2[:n_bags], dY[i, :n_bags], lr)
    pipe.ctx.check()
    assert torch.equal(W_hot, W_std)
    assert torch.equal(Y, Y2)
    ref = _prep_ref(ds, 5.0, 3, "t", t=c.t, small=small, dim=c.dim)
    Wr = oracle.extract(W, ref["remap"], ref["H"])
    pk = ref["pack"]
    Tn = c.n_tables
    for i in range(nb):
        b = first + i
        r0, r1 = b * c.batch, min((b + 1) * c.batch, pk["n_hot"])
        n_bags = (r1 - r0) * Tn
        bi = pk["hot_idx"][r0 * Tn: r1 * Tn]
        if i == nb - 1:   # the last trained batch's forward output
            Yref, _ = oracle.emb_fwd(Wr, bi, None, 1, n_bags)
            ok, worst = close(Y[:n_bags].cpu().numpy(), Yref)
            assert ok, worst
        Wr, _ = oracle.emb_bwd_sgd(Wr, bi, None, 1, n_bags, dY[i, :n_bags].cpu(), lr)
    ok, worst = close(W_hot.cpu().numpy(), Wr)
    assert ok, worst
