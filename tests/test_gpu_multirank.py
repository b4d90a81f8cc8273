"""G > 1 parity on ONE GPU: "virtual ranks" (fae_comm_init_loopback, test-only).

W ctxs in this process, one host thread and one CUDA stream each, form a
loopback group: every collective of libfae (the sharded profile's select
histograms, candidates, loggers and T; the a11 count / payload all-gathers)
runs as a host rendezvous plus device copies instead of NCCL, and everything
else is the library's multi-rank code path.  Checked against the oracle
(SURVEY §8(c) O10 "sharding invariance"):

* the sharded fae_profile selects exactly oracle.sample over the global
  record ids, and its loggers / T equal oracle.histogram of the whole dataset
  (bit-exact), at a size that takes two radix-select levels;
* fae_sync_hot_grads returns the global sparse sum (sorted, rank-order sums,
  identical bits on every rank) within 1e-6 + 1e-5|ref| of an fp64 sum;
* fae_emb_bwd_update with a comm and fae_train_hot_batches over W ranks ==
  the oracle's sequential SGD over the GLOBAL batches (global batch i = the
  concatenation, in rank order, of each rank's hot batch i; P:L217-220,
  L298-301, L757-758 weak scaling), within tolerance, and the W replicas are
  bit-identical.
"""
import threading

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


_KEY = [1000]

# Kaggle-shaped (26 tables, the same skew of sizes, D = 16, B = 2048) with
# rows / 100, so each virtual rank's full table fits beside the others
KAGGLE_SMALL = gen.Config("kaggle-small", [max(3, r // 100) for r in gen.KAGGLE_ROWS], 16, 2048, 1,
                          records=200_000, t=1e-6)


# Alibaba-shaped multi-hot (pooling U{20..100}) with a small batch, so a
# 24k-record run has several hot batches per rank
ALI_SMALL = gen.Config("ali-small", gen.ALIBABA_ROWS, 16, 128, 0, 20, 100, records=24_000, t=1e-7)


def config(name):
    return {"kaggle-small": KAGGLE_SMALL, "ali-small": ALI_SMALL}.get(name) or gen.CONFIGS[name]


def test_gen_device_equals_cpu():
    """The seeded generators draw the same bits on the GPU as on the CPU (the
    virtual ranks generate their shards on the device, the oracle on the host),
    including the 10M-row Zipf tables and variable pooling."""
    dev = torch.device("cuda", 0)
    for name, n, base in (("kaggle", 3000, 12345), ("alibaba", 500, 77)):
        c = gen.CONFIGS[name]
        a = gen.make_dataset(c, n_records=n, seed=5, record_base=base)
        b = gen.make_dataset(c, n_records=n, seed=5, record_base=base, device=dev)
        assert torch.equal(a.idx, b.idx.cpu())
        if a.off is not None:
            assert torch.equal(a.off, b.off.cpu())
    assert torch.equal(gen.make_weights(1000, 16), gen.make_weights(1000, 16, device=dev).cpu())


def run_ranks(world, body, timeout=600):
    """body(rank, stream) in `world` threads (one per virtual rank); returns
    the per-rank results, re-raising the first failure."""
    _KEY[0] += 1
    key = _KEY[0]
    out, errs = [None] * world, []

    def th(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream(device=0)
            with torch.cuda.stream(s):
                out[r] = body(r, s, key)
                s.synchronize()
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))

    ts = [threading.Thread(target=th, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert not any(t.is_alive() for t in ts), "virtual ranks hung"
    if errs:
        raise errs[0][1]
    return out


@pytest.fixture(autouse=True)
def _loopback(monkeypatch):
    monkeypatch.setenv("FAE_LOOPBACK", "1")


def _pipe(cfg, world, rank, stream, key):
    from paper_2103_00686_b200.pipeline import FaePipeline
    pipe = FaePipeline(cfg.rows, cfg.dim, cfg.batch, cfg.pool, max_pool=max(cfg.pool_hi, 1),
                       max_world=world)
    pipe.ctx.set_stream(stream)
    fae().fae_comm_init_loopback(pipe.ctx, key, rank, world)
    return pipe


def test_loopback_needs_env(monkeypatch):
    monkeypatch.delenv("FAE_LOOPBACK")
    m = fae()
    ctx = m.fae_create(0, max_tables=1, max_rows=10, max_batch_lookups=16, max_batch_bags=16,
                       max_dim=16, max_world=2)
    with pytest.raises(m.FaeError) as e:
        m.fae_comm_init_loopback(ctx, 1, 0, 2)
    assert e.value.name == "INVALID_ARG"


# ----------------------------------------------------------------------------
# a1 + a2 sharded: the global sample and loggers
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("world,cfgname,R,x", [(2, "tiny", 2_400_000, 5.0),    # two select levels
                                               (4, "tiny", 2_400_000, 5.0),
                                               (8, "tiny", 2_400_000, 5.0),
                                               (3, "alibaba", 30_000, 5.0),    # offsets, ragged shards
                                               (4, "kaggle", 200_000, 100.0)])
def test_sharded_profile_equals_unsharded_oracle(world, cfgname, R, x):
    m = fae()
    cfg = gen.CONFIGS[cfgname]
    seed = 4242
    full = gen.make_dataset(cfg, n_records=R, seed=17)
    samp_ref = oracle.sample(R, x, seed)
    counts_ref, T_ref, st = oracle.histogram(full.rows, full.idx, full.off, full.fixed_pool, R, samp_ref)
    assert st == 0
    # contiguous shards, the last one ragged
    per = -(-R // world)
    bounds = [(min(r * per, R), min((r + 1) * per, R)) for r in range(world)]
    dev = torch.device("cuda", 0)

    def body(rank, s, key):
        lo, hi = bounds[rank]
        ds = gen.make_dataset(cfg, n_records=hi - lo, seed=17, device=dev, record_base=lo)
        pipe = _pipe(cfg, world, rank, s, key)
        counts = torch.empty(sum(cfg.rows), dtype=torch.int32, device=dev)
        samp = torch.empty(max(hi - lo, 1), dtype=torch.int64, device=dev)
        T, ns = m.fae_profile(pipe.ctx, cfg.rows, cfg.dim, ds.idx, ds.off, ds.fixed_pool, hi - lo, x,
                              seed, counts, samp, record_base=lo, n_records_global=R)
        return (samp[:ns].cpu().numpy() + lo, counts.cpu().numpy().view(np.uint32), T)

    res = run_ranks(world, body)
    ids = np.concatenate([r[0] for r in res])
    assert np.array_equal(ids, samp_ref)                  # global sample, ascending
    for _, counts, T in res:
        assert np.array_equal(counts, counts_ref)         # loggers summed over ranks
        assert list(T) == list(T_ref)


# ----------------------------------------------------------------------------
# a11 on a caller-visible sparse gradient
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sync_hot_grads_global_sum(world):
    m = fae()
    H, D, cap = 5000, 16, 4096 * 8
    rng = np.random.default_rng(world)
    lists = []
    for r in range(world):
        n = int(rng.integers(0 if r == 1 else 1, 3000))   # rank 1 may contribute nothing
        rows = np.sort(rng.choice(H, n, replace=False)).astype(np.int32)
        vals = rng.uniform(-1, 1, (n, D)).astype(np.float32)
        lists.append((rows, vals))
    ref = {}
    for rows, vals in lists:                               # fp64 sum over ranks
        for x, v in zip(rows, vals):
            ref[int(x)] = ref.get(int(x), 0.0) + v.astype(np.float64)
    ref_rows = np.array(sorted(ref), np.int32)
    ref_vals = np.stack([ref[int(x)] for x in ref_rows]) if len(ref_rows) else np.zeros((0, D))
    dev = torch.device("cuda", 0)

    def body(rank, s, key):
        ctx = m.fae_create(0, max_tables=1, max_rows=H, max_batch_lookups=4096, max_batch_bags=4096,
                           max_dim=D, max_world=world)
        ctx.set_stream(s)
        m.fae_comm_init_loopback(ctx, key, rank, world)
        rows, vals = lists[rank]
        R = torch.zeros(cap, dtype=torch.int32, device=dev)
        V = torch.zeros(cap, D, device=dev)
        R[:len(rows)] = torch.from_numpy(rows).to(dev)
        V[:len(rows)] = torch.from_numpy(vals).to(dev)
        n = m.fae_sync_hot_grads(ctx, R, V, len(rows))
        return R[:n].cpu().numpy(), V[:n].cpu().numpy()

    res = run_ranks(world, body)
    for rows, vals in res:
        assert np.array_equal(rows, ref_rows)
        ok, worst = close(vals, ref_vals)
        assert ok, worst
        assert np.array_equal(vals, res[0][1])             # identical bits on every rank


# ----------------------------------------------------------------------------
# the training loop at W ranks vs O10 (global batches)
# ----------------------------------------------------------------------------
def _global_batches(cfg, per_rank_packs, nb):
    """Global batch i = concat over ranks of rank r's hot batch i (rank order);
    returns [(idx, off, P, n_bags, [(rank, bag0, n_bags_r)])]."""
    B, Tn = cfg.batch, cfg.n_tables
    out = []
    for i in range(nb):
        idx_parts, off_parts, segs, nbags = [], [], [], 0
        for r, pk in enumerate(per_rank_packs):
            r0, r1 = i * B, min((i + 1) * B, pk["n_hot"])
            if r1 <= r0:
                continue
            n_b = (r1 - r0) * Tn
            if cfg.pool > 0:
                P = cfg.pool
                idx_parts.append(pk["hot_idx"][r0 * Tn * P: r1 * Tn * P])
            else:
                o = pk["hot_off"][r0 * Tn: r1 * Tn + 1]
                idx_parts.append(pk["hot_idx"][o[0]:o[-1]])
                off_parts.append(np.diff(o))
            segs.append((r, nbags, n_b))
            nbags += n_b
        idx = np.concatenate(idx_parts) if idx_parts else np.zeros(0, np.int32)
        if cfg.pool > 0:
            off, P = None, cfg.pool
        else:
            off = np.concatenate([[0], np.cumsum(np.concatenate(off_parts))]).astype(np.int64)
            P = 0
        out.append((idx, off, P, nbags, segs))
    return out


def _oracle_prep(cfg, full, R, x, seed, t, small):
    samp = oracle.sample(R, x, seed)
    counts, T, _ = oracle.histogram(full.rows, full.idx, full.off, full.fixed_pool, R, samp)
    kmin = oracle.kmin_fixed_t(full.rows, cfg.dim, small, T, t, x)
    hot = oracle.tag_rows(full.rows, cfg.dim, small, counts, kmin)
    return oracle.remap(full.rows, hot)


@pytest.mark.parametrize("world,cfgname,R,t,small,standalone,table", [
    (2, "kaggle-small", 200_000, 1e-5, 1 << 20, False, None),   # merge by binary search
    (2, "kaggle-small", 200_000, 1e-5, 1 << 20, False, "1"),    # merge by row-position table
    (4, "kaggle-small", 200_000, 1e-5, 1 << 20, False, None),   # table (default above 2 ranks)
    (4, "kaggle-small", 200_000, 1e-5, 1 << 20, False, "0"),
    (8, "tiny", 40_000, 1e-2, 0, False, None),
    (3, "ali-small", 24_000, 1e-7, 1 << 20, False, None),
    (4, "tiny", 20_000, 1e-2, 0, True, None),            # fae_emb_fwd + fae_emb_bwd_update with a comm
])
def test_train_world_equals_oracle_global_batches(world, cfgname, R, t, small, standalone, table, monkeypatch):
    m = fae()
    if table is not None:
        monkeypatch.setenv("FAE_MERGE_TABLE", table)   # read at fae_create
    cfg = config(cfgname)
    x, seed, lr = 5.0, 3, 0.05
    full = gen.make_dataset(cfg, n_records=R, seed=23)
    rm, base, H = _oracle_prep(cfg, full, R, x, seed, t, small)
    W0 = gen.make_weights(sum(cfg.rows), cfg.dim)
    W_hot0 = oracle.extract(W0, rm, H)
    per = R // world                                       # equal shards (weak scaling)
    S = cfg.batch * cfg.n_tables
    n_steps = 6
    dev = torch.device("cuda", 0)
    packs = []
    for r in range(world):                                 # oracle per-shard classification
        sl = gen.make_dataset(cfg, n_records=per, seed=23, record_base=r * per)
        flag = oracle.classify(sl.rows, sl.idx, sl.off, sl.fixed_pool, per, rm)
        packs.append(oracle.pack(sl.rows, sl.idx, sl.off, sl.fixed_pool, per, rm, flag))
    nb = min(n_steps, max(-(-p["n_hot"] // cfg.batch) for p in packs))
    assert nb >= 2
    dYs = [gen.make_dy(nb * S, cfg.dim, seed=300 + r).view(nb, S, cfg.dim) for r in range(world)]

    def body(rank, s, key):
        ds = gen.make_dataset(cfg, n_records=per, seed=23, device=dev, record_base=rank * per)
        pipe = _pipe(cfg, world, rank, s, key)
        prep = pipe.preprocess(ds.idx, ds.off, per, x_pct=x, seed=seed, t=t, small_table_bytes=small,
                               record_base=rank * per, n_records_global=world * per)
        W_hot = pipe.extract(W0.to(dev), prep).clone()
        dY = dYs[rank].to(dev)
        Y = torch.zeros(S, cfg.dim, device=dev)
        if standalone:
            nb_local = prep.packed["n_hot_batches"]
            for i in range(nb):
                if i < nb_local:
                    idx, off, n_bags = pipe.batch_args(prep, i)
                else:
                    idx, off, n_bags = prep.hot_idx[:0], None, 0
                m.fae_emb_fwd(pipe.ctx, W_hot, idx, off, pipe.pool, n_bags, Y[:n_bags])
                m.fae_emb_bwd_update(pipe.ctx, W_hot, idx, off, pipe.pool, n_bags, dY[i, :n_bags], lr)
        else:
            pipe.group(prep)
            pipe.train(W_hot, 0, nb, dY, Y, lr)
        pipe.ctx.check()
        return W_hot.cpu().numpy(), prep.packed

    res = run_ranks(world, body)
    for r in range(world):                                 # per-shard classification bit-exact
        assert res[r][1]["n_hot"] == packs[r]["n_hot"]
    for r in range(1, world):                              # replicas bit-identical
        assert np.array_equal(res[r][0], res[0][0]), f"rank {r} replica differs"
    Wr = W_hot0
    for i, (idx, off, P, nbags, segs) in enumerate(_global_batches(cfg, packs, nb)):
        dY = np.concatenate([dYs[r][i, :n_b].numpy() for r, _, n_b in segs]) if segs else \
            np.zeros((0, cfg.dim), np.float32)
        Wr, st = oracle.emb_bwd_sgd(Wr, idx, off, P, nbags, dY, lr)
        assert st == 0
    ok, worst = close(res[0][0], Wr)
    assert ok, worst


# ----------------------------------------------------------------------------
# NEXT-2 at G > 1: the DLRM hot step with the MLP gradient all-reduce fused
# with the hot-gradient exchange
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("world,R", [(2, 12_000), (3, 12_000)])
def test_train_dlrm_world_equals_oracle_global_batches(world, R):
    """fae_train_dlrm_batches over `world` virtual ranks == the oracle's DLRM
    trained on the GLOBAL batches (global batch i = the concatenation, in
    rank order, of each rank's hot batch i; loss = mean over the global
    batch), hot rows and MLP parameters identical on every rank (pedantic
    fp32 GEMMs)."""
    from oracle import dlrm as odlrm
    m = fae()
    cfg = gen.CONFIGS["tiny"]
    x, seed, t, small = 5.0, 3, 1e-2, 0
    Tn, D, B = cfg.n_tables, cfg.dim, cfg.batch
    full = gen.make_dataset(cfg, n_records=R, seed=23)
    rm, base, H = _oracle_prep(cfg, full, R, x, seed, t, small)
    W0 = gen.make_weights(sum(cfg.rows), D)
    per = R // world
    n_dense, bottom, top = 4, [12, D], [20, 1]
    dims = gen.dlrm_dims(n_dense, bottom, top, Tn, D)
    p0 = gen.make_dlrm_params(dims, seed=41)
    dense_all = gen.make_dense(R, n_dense)
    label_all = gen.make_labels(R, n_dense)
    packs = []
    for r in range(world):
        sl = gen.make_dataset(cfg, n_records=per, seed=23, record_base=r * per)
        flag = oracle.classify(sl.rows, sl.idx, sl.off, sl.fixed_pool, per, rm)
        packs.append(oracle.pack(sl.rows, sl.idx, sl.off, sl.fixed_pool, per, rm, flag))
    nb = min(4, max(-(-p["n_hot"] // B) for p in packs))
    assert nb >= 2
    lr_mlp, lr_emb = 0.05, 0.01
    dev = torch.device("cuda", 0)

    def body(rank, s, key):
        ds = gen.make_dataset(cfg, n_records=per, seed=23, device=dev, record_base=rank * per)
        pipe = _pipe(cfg, world, rank, s, key)
        prep = pipe.preprocess(ds.idx, ds.off, per, x_pct=x, seed=seed, t=t, small_table_bytes=small,
                               record_base=rank * per, n_records_global=world * per)
        W_hot = pipe.extract(W0.to(dev), prep).clone()
        pipe.group(prep)
        model = m.Dlrm(pipe.ctx, n_dense, bottom, top, Tn, D, B, tf32=False)
        params = gen.dlrm_pad(p0, dims).to(dev)
        model.train_batches(params, W_hot, 0, nb, prep.hot_ids, dense_all[rank * per:(rank + 1) * per].to(dev),
                            label_all[rank * per:(rank + 1) * per].to(dev), lr_mlp, lr_emb)
        pipe.ctx.check()
        return W_hot.cpu().numpy(), gen.dlrm_unpad(params.cpu(), dims).numpy()

    res = run_ranks(world, body)
    for r in range(1, world):
        assert np.array_equal(res[r][0], res[0][0]), f"rank {r} hot table differs"
        assert np.array_equal(res[r][1], res[0][1]), f"rank {r} MLP parameters differ"
    Wr = oracle.extract(W0, rm, H)
    p = p0.double().numpy()
    dn, lb = dense_all.double().numpy(), label_all.double().numpy()
    for i, (idx, off, P, nbags, segs) in enumerate(_global_batches(cfg, packs, nb)):
        recs = np.concatenate([packs[r]["hot_ids"][i * B: i * B + n_b // Tn] + r * per for r, _, n_b in segs])
        Yb, st = oracle.emb_fwd(Wr, idx, off, P, nbags)
        assert st == 0
        L, cache = odlrm.forward(p, dims, len(bottom), dn[recs], Yb.reshape(-1, Tn, D).astype(np.float64), lb[recs])
        p, dYb, _ = odlrm.backward_sgd(p, dims, len(bottom), cache, lr_mlp)
        Wr, st = oracle.emb_bwd_sgd(Wr, idx, off, P, nbags, dYb.reshape(nbags, D).astype(np.float32), lr_emb)
        assert st == 0
    got_p = res[0][1].astype(np.float64)
    assert np.all(np.abs(got_p - p) <= 1e-6 + 1e-5 * np.abs(p)), np.abs(got_p - p).max()
    ok, worst = close(res[0][0], Wr)
    assert ok, worst
