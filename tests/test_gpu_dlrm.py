"""NEXT-2 parity: the DLRM hot step (libfae fae_dlrm_*, cuBLAS GEMMs + hand
written kernels) against the fp64 oracle (oracle/dlrm.py, pinned by
tests/test_dlrm_oracle.py).

Tolerances (R34): pedantic fp32 GEMMs — loss within 1e-5
relative, every updated parameter within 1e-6 + 1e-5|ref| (north_star's fp32
bound), dY within 1e-5 max|dY| + 1e-4|ref| (chains of <= 3 fp32 GEMMs of
K <= 64); TF32 tensor-core GEMMs (10-bit mantissa, unit roundoff 2^-11) —
loss within 1e-3 relative, parameter updates within 2% of the largest
update, dY within 2% of max|dY|."""
import numpy as np
import pytest
import torch

import gen
import oracle
from oracle import dlrm as odlrm

pytestmark = pytest.mark.gpu


def fae():
    import paper_2103_00686_b200 as m
    return m


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def _ctx(rows, dim, lookups, bags):
    m = fae()
    return m.fae_create(0, max_tables=len(rows), max_rows=sum(rows), max_batch_lookups=lookups,
                        max_batch_bags=bags, max_dim=dim, max_world=1)


@pytest.mark.parametrize("tf32", [False, True])
@pytest.mark.parametrize("B,maxB", [(37, 64), (64, 64), (1, 8)])
def test_dlrm_step_equals_oracle(dev, tf32, B, maxB):
    m = fae()
    n_dense, bottom, top, Tn, D = 5, [16, 8], [24, 12, 1], 3, 8
    ctx = _ctx([100] * Tn, D, 1024, 1024)
    model = m.Dlrm(ctx, n_dense, bottom, top, Tn, D, maxB, tf32=tf32)
    dims = gen.dlrm_dims(n_dense, bottom, top, Tn, D)
    assert model.n_params == sum((i + 3) // 4 * 4 * o + o for i, o in dims)
    p0 = gen.make_dlrm_params(dims, seed=11)
    dense = gen.make_dense(B, n_dense, seed=12)
    label = gen.make_labels(B, n_dense, seed=13)
    Y = (0.5 * gen.make_dy(B * Tn, D, seed=14)).view(B, Tn, D)
    lr = 0.1
    params = gen.dlrm_pad(p0, dims).to(dev)
    dY = torch.zeros(B, Tn, D, device=dev)
    model.step(params, B, dense.to(dev), label.to(dev), Y.to(dev), dY, lr, train=True)
    s, n = model.loss()
    L, cache = odlrm.forward(p0.double().numpy(), dims, len(bottom), dense.double().numpy(),
                             Y.double().numpy(), label.double().numpy())
    newp, dYr, _ = odlrm.backward_sgd(p0.double().numpy(), dims, len(bottom), cache, lr)
    assert n == B
    got_p, got_dy = gen.dlrm_unpad(params.cpu(), dims).double().numpy(), dY.cpu().double().numpy()
    if not tf32:
        assert abs(s / B - L) <= 1e-5 * abs(L)
        assert np.all(np.abs(got_p - newp) <= 1e-6 + 1e-5 * np.abs(newp))
        sc = np.abs(dYr).max()
        assert np.all(np.abs(got_dy - dYr) <= 1e-5 * sc + 1e-4 * np.abs(dYr))
    else:
        assert abs(s / B - L) <= 1e-3 * abs(L)
        upd = np.abs(newp - p0.double().numpy()).max()
        assert np.abs(got_p - newp).max() <= 0.02 * upd + 1e-7
        assert np.abs(got_dy - dYr).max() <= 0.02 * np.abs(dYr).max()
    # forward only: loss of the updated model, parameters untouched
    before = params.clone()
    model.step(params, B, dense.to(dev), label.to(dev), Y.to(dev), None, 0.0, train=False)
    s2, n2 = model.loss()
    L2, _ = odlrm.forward(newp, dims, len(bottom), dense.double().numpy(), Y.double().numpy(),
                          label.double().numpy())
    assert n2 == B and abs(s2 / B - L2) <= (1e-5 if not tf32 else 1e-3) * abs(L2)
    assert torch.equal(before, params)


def test_dlrm_bad_config(dev):
    m = fae()
    ctx = _ctx([100], 8, 64, 64)
    with pytest.raises(m.FaeError):
        m.Dlrm(ctx, 5, [16, 4], [8, 1], 1, 8, 16)          # bottom output != D
    with pytest.raises(m.FaeError):
        m.Dlrm(ctx, 5, [16, 8], [8, 2], 1, 8, 16)          # top output != 1


@pytest.mark.parametrize("cfgname,R,t,small,exchange", [("tiny", 10_000, 1e-2, 0, False),
                                                       ("tiny", 10_000, 1e-2, 0, True)])
def test_train_dlrm_batches_equals_oracle(dev, cfgname, R, t, small, exchange, monkeypatch):
    """The full hot step over grouped hot batches (a8 of the grouped loop ->
    DLRM forward/backward/SGD -> a9 + a10, one captured graph) == the oracle
    sequence: emb_fwd, the fp64 DLRM, emb_bwd_sgd with its dY, batch after
    batch (pedantic fp32 GEMMs).  exchange: the data-parallel path (MLP
    gradient all-reduce fused with the hot-gradient all-gathers, captured
    with NCCL) on a 1-rank communicator."""
    m = fae()
    from paper_2103_00686_b200.pipeline import FaePipeline
    monkeypatch.setenv("FAE_FORCE_MERGE", "1" if exchange else "0")   # read at fae_create
    c = gen.CONFIGS[cfgname]
    ds = gen.make_dataset(c, n_records=R, seed=5)
    dd = ds.to(dev)
    Tn, D, B = c.n_tables, c.dim, c.batch
    pipe = FaePipeline(ds.rows, D, B, c.pool)
    if exchange:
        m.fae_comm_init(pipe.ctx, m.fae_get_nccl_id(), 0, 1)
    prep = pipe.preprocess(dd.idx, dd.off, R, x_pct=5.0, seed=3, t=t, small_table_bytes=small)
    W = gen.make_weights(sum(ds.rows), D)
    W_hot = pipe.extract(W.to(dev), prep).clone()
    pipe.group(prep)
    n_dense, bottom, top = 4, [12, D], [20, 1]
    dims = gen.dlrm_dims(n_dense, bottom, top, Tn, D)
    model = m.Dlrm(pipe.ctx, n_dense, bottom, top, Tn, D, B, tf32=False)
    p0 = gen.make_dlrm_params(dims, seed=21)
    params = gen.dlrm_pad(p0, dims).to(dev)
    dense = gen.make_dense(R, n_dense, seed=22)
    label = gen.make_labels(R, n_dense, seed=23)
    nb = min(prep.packed["n_hot_batches"], 5)
    assert nb >= 3
    lr_mlp, lr_emb = 0.05, 0.01
    model.train_batches(params, W_hot, 0, nb, prep.hot_ids, dense.to(dev), label.to(dev), lr_mlp, lr_emb)
    s, n = model.loss()
    pipe.ctx.check()
    # oracle
    ref = oracle
    samp = ref.sample(R, 5.0, 3)
    counts, T, _ = ref.histogram(ds.rows, ds.idx, None, 1, R, samp)
    kmin = ref.kmin_fixed_t(ds.rows, D, small, T, t, 5.0)
    hot = ref.tag_rows(ds.rows, D, small, counts, kmin)
    rm, base, H = ref.remap(ds.rows, hot)
    flag = ref.classify(ds.rows, ds.idx, None, 1, R, rm)
    pk = ref.pack(ds.rows, ds.idx, None, 1, R, rm, flag)
    Wr = ref.extract(W, rm, H)
    p = p0.double().numpy()
    dn, lb = dense.double().numpy(), label.double().numpy()
    Ltot, ntot = 0.0, 0
    for i in range(nb):
        r0, r1 = i * B, min((i + 1) * B, pk["n_hot"])
        recs = pk["hot_ids"][r0:r1]
        nbags = (r1 - r0) * Tn
        bi = pk["hot_idx"][r0 * Tn: r1 * Tn]
        Yb, st = ref.emb_fwd(Wr, bi, None, 1, nbags)
        assert st == 0
        L, cache = odlrm.forward(p, dims, len(bottom), dn[recs], Yb.reshape(-1, Tn, D).astype(np.float64), lb[recs])
        Ltot += L * (r1 - r0)
        ntot += r1 - r0
        p, dYb, _ = odlrm.backward_sgd(p, dims, len(bottom), cache, lr_mlp)
        Wr, st = ref.emb_bwd_sgd(Wr, bi, None, 1, nbags, dYb.reshape(nbags, D).astype(np.float32), lr_emb)
        assert st == 0
    assert n == ntot
    assert abs(s - Ltot) <= 1e-5 * abs(Ltot)
    got_p = gen.dlrm_unpad(params.cpu(), dims).double().numpy()
    assert np.all(np.abs(got_p - p) <= 1e-6 + 1e-5 * np.abs(p)), np.abs(got_p - p).max()
    got_w = W_hot.cpu().double().numpy()
    assert np.all(np.abs(got_w - Wr) <= 1e-6 + 1e-5 * np.abs(Wr)), np.abs(got_w - Wr).max()


def _trainer(dev, R, n_test, r_start, tf32=False):
    m = fae()
    from paper_2103_00686_b200.pipeline import FaePipeline, FaeTrainer, MixedEpoch
    c = gen.CONFIGS["tiny"]
    ds = gen.make_dataset(c, n_records=R, seed=5)
    dd = ds.to(dev)
    Tn, D, B = c.n_tables, c.dim, c.batch
    pipe = FaePipeline(ds.rows, D, B, c.pool)
    prep = pipe.preprocess(dd.idx, dd.off, R, x_pct=5.0, seed=3, t=1e-2, small_table_bytes=0)
    W = gen.make_weights(sum(ds.rows), D).to(dev)
    W_hot = pipe.extract(W, prep).clone()
    ep = MixedEpoch(pipe, prep, W, dd.idx, dd.off, R, W_hot)
    n_dense, bottom, top = 4, [12, D], [20, 1]
    dims = gen.dlrm_dims(n_dense, bottom, top, Tn, D)
    params = gen.dlrm_pad(gen.make_dlrm_params(dims, seed=31), dims).to(dev)
    dense = gen.make_dense(R, n_dense).to(dev)
    label = gen.make_labels(R, n_dense).to(dev)
    # held-out records: the next n_test records of the stream, global row ids
    tds = gen.make_dataset(c, n_records=n_test, seed=5, record_base=R)
    base = np.concatenate([[0], np.cumsum(ds.rows)])[:Tn]
    tidx = torch.from_numpy((tds.idx.numpy().reshape(n_test, Tn) + base).reshape(-1).astype(np.int32)).to(dev)
    tdense = gen.make_dense(n_test, n_dense, record_base=R).to(dev)
    tlabel = gen.make_labels(n_test, n_dense, record_base=R).to(dev)
    tr = FaeTrainer(ep, n_dense, bottom, top, params, dense, label, tidx, None, n_test, tdense, tlabel, tf32=tf32)
    sched = m.Scheduler(ep.n_cold_batches, ep.n_hot_batches, r_start)
    return dict(tr=tr, ep=ep, sched=sched, ds=ds, prep=prep, W0=gen.make_weights(sum(ds.rows), D), dims=dims,
                p0=gen.make_dlrm_params(dims, seed=31), dense=dense.cpu(), label=label.cpu(), tds=tds,
                tdense=tdense.cpu(), tlabel=tlabel.cpu(), bottom=bottom)


def test_fae_trainer_epoch_equals_oracle(dev):
    """NEXT-2 + NEXT-3 end to end: one epoch of FAE training of the DLRM in
    the scheduler's order (cold first, R(100): all cold, swap, all hot),
    cold batches on the master tables, hot on the replica, the post-swap test
    loss on held-out records == the oracle sequence (fp64 DLRM, emb fwd /
    bwd+SGD, scatter / extract at the swaps, the test loss over the held-out
    records), pedantic fp32 GEMMs."""
    t = _trainer(dev, 3000, 256, 100.0)
    tr, ep, sched = t["tr"], t["ep"], t["sched"]
    log = []
    lr_mlp, lr_emb = 0.05, 0.01
    phases = tr.run_epoch(sched, lr_mlp, lr_emb, log)
    ep.finish()
    tr.ep.pipe.ctx.check()
    ep.cold.ctx.check()
    assert [k for k, _, _ in phases] == ["cold", "hot"] and sched.swaps == 1 and len(log) == 1
    # oracle
    ds, c = t["ds"], gen.CONFIGS["tiny"]
    Tn, D, B, R = c.n_tables, c.dim, c.batch, 3000
    samp = oracle.sample(R, 5.0, 3)
    counts, T, _ = oracle.histogram(ds.rows, ds.idx, None, 1, R, samp)
    kmin = oracle.kmin_fixed_t(ds.rows, D, 0, T, 1e-2, 5.0)
    rm, base, H = oracle.remap(ds.rows, oracle.tag_rows(ds.rows, D, 0, counts, kmin))
    pk = oracle.pack(ds.rows, ds.idx, None, 1, R, rm, oracle.classify(ds.rows, ds.idx, None, 1, R, rm))
    gbase = np.concatenate([[0], np.cumsum(ds.rows)])[:Tn]
    Wf = t["W0"].numpy().copy()
    p = t["p0"].double().numpy()
    dn, lb = t["dense"].double().numpy(), t["label"].double().numpy()
    nb_ = len(t["bottom"])
    dims = t["dims"]

    def step(Wt, idx_rows, recs, p):
        nbags = len(recs) * Tn
        Yb, _ = oracle.emb_fwd(Wt, idx_rows, None, 1, nbags)
        L, cache = odlrm.forward(p, dims, nb_, dn[recs], Yb.reshape(-1, Tn, D).astype(np.float64), lb[recs])
        p, dYb, _ = odlrm.backward_sgd(p, dims, nb_, cache, lr_mlp)
        Wt, _ = oracle.emb_bwd_sgd(Wt, idx_rows, None, 1, nbags, dYb.reshape(nbags, D).astype(np.float32), lr_emb)
        return Wt, p

    ids = ds.idx.numpy().reshape(R, Tn)
    for i in range(-(-pk["n_cold"] // B)):                   # cold phase on the master tables
        recs = pk["cold_ids"][i * B:(i + 1) * B]
        Wf, p = step(Wf, (ids[recs] + gbase).reshape(-1).astype(np.int32), recs, p)
    # swap: the held-out test loss on the master tables (the replica is current in Wf)
    tids = (t["tds"].idx.numpy().reshape(-1, Tn) + gbase).reshape(-1).astype(np.int32)
    Yt, _ = oracle.emb_fwd(Wf, tids, None, 1, len(tids))
    Lt, _ = odlrm.forward(p, dims, nb_, t["tdense"].double().numpy(), Yt.reshape(-1, Tn, D).astype(np.float64),
                          t["tlabel"].double().numpy())
    assert abs(log[0]["test_loss"] - Lt) <= 1e-5 * abs(Lt)
    Wh = oracle.extract(Wf, rm, H)
    for i in range(-(-pk["n_hot"] // B)):                    # hot phase on the replica
        r0, r1 = i * B, min((i + 1) * B, pk["n_hot"])
        Wh, p = step(Wh, pk["hot_idx"][r0 * Tn: r1 * Tn], pk["hot_ids"][r0:r1], p)
    Wf = oracle.scatter_hot(Wf, Wh, rm)
    got_p = gen.dlrm_unpad(tr.params.cpu(), t["dims"]).double().numpy()
    assert np.all(np.abs(got_p - p) <= 1e-6 + 1e-5 * np.abs(p)), np.abs(got_p - p).max()
    got_w = ep.W.cpu().double().numpy()
    assert np.all(np.abs(got_w - Wf) <= 1e-6 + 1e-5 * np.abs(Wf)), np.abs(got_w - Wf).max()


def test_fae_trainer_scheduler_invariants(dev):
    """R(50) start with loss feedback: every batch of both kinds trained once,
    cold first, one test loss per swap, rates in [1, 100], deterministic."""
    outs = []
    for _ in range(2):
        t = _trainer(dev, 6000, 256, 50.0, tf32=True)
        tr, ep, sched = t["tr"], t["ep"], t["sched"]
        log = []
        phases = tr.run_epoch(sched, 0.05, 0.01, log)
        ep.finish()
        seen = {"cold": [], "hot": []}
        for k, f, n in phases:
            seen[k].extend(range(f, f + n))
        assert seen["cold"] == list(range(ep.n_cold_batches)) and seen["hot"] == list(range(ep.n_hot_batches))
        assert phases[0][0] == "cold" and len(log) == sched.swaps >= 1
        assert all(1.0 <= e["rate"] <= 100.0 and np.isfinite(e["test_loss"]) for e in log)
        outs.append((tr.params.cpu(), ep.W.cpu(), [e["test_loss"] for e in log]))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1]) and outs[0][2] == outs[1][2]


@pytest.mark.parametrize("model,tf32", [("rmc2", False), ("rmc2", True), ("rmc3", True)])
def test_dlrm_step_paper_shapes(dev, model, tf32):
    """One DLRM step at the paper's shapes (tab:benchmarks P:L516-526: RMC2
    13-512-256-64-16 / 512-256-1, D 16, B 2048; RMC3 13-512-256-64 /
    512-512-256-1, D 64, B 4096; 26 sparse features) against the fp64
    oracle, with the tolerances of the module docstring."""
    m = fae()
    n_dense, bottom, top, D, B = ((13, [512, 256, 64, 16], [512, 256, 1], 16, 2048) if model == "rmc2" else
                                  (13, [512, 256, 64], [512, 512, 256, 1], 64, 4096))
    Tn = 26
    ctx = _ctx([1000] * Tn, D, B * Tn, B * Tn)
    mdl = m.Dlrm(ctx, n_dense, bottom, top, Tn, D, B, tf32=tf32)
    dims = gen.dlrm_dims(n_dense, bottom, top, Tn, D)
    p0 = gen.make_dlrm_params(dims, seed=51)
    dense = gen.make_dense(B, n_dense, seed=52)
    label = gen.make_labels(B, n_dense, seed=53)
    Y = (0.05 * gen.make_dy(B * Tn, D, seed=54)).view(B, Tn, D)
    lr = 0.05
    params = gen.dlrm_pad(p0, dims).to(dev)
    dY = torch.zeros(B, Tn, D, device=dev)
    mdl.step(params, B, dense.to(dev), label.to(dev), Y.to(dev), dY, lr, train=True)
    s, n = mdl.loss()
    L, cache = odlrm.forward(p0.double().numpy(), dims, len(bottom), dense.double().numpy(), Y.double().numpy(),
                             label.double().numpy())
    newp, dYr, _ = odlrm.backward_sgd(p0.double().numpy(), dims, len(bottom), cache, lr)
    got_p = gen.dlrm_unpad(params.cpu(), dims).double().numpy()
    got_dy = dY.cpu().double().numpy()
    assert n == B
    if not tf32:
        assert abs(s / B - L) <= 1e-5 * abs(L)
        assert np.all(np.abs(got_p - newp) <= 1e-6 + 1e-5 * np.abs(newp)), np.abs(got_p - newp).max()
        sc = np.abs(dYr).max()
        assert np.all(np.abs(got_dy - dYr) <= 1e-5 * sc + 1e-4 * np.abs(dYr))
    else:
        # TF32 (R34): inputs rounded to a 10-bit mantissa, u = 2^-11; a K-term
        # dot product of random-sign terms errs by ~2u*sqrt(K) relative, and
        # dY is len(top) chained GEMMs deep in the backward (K <= 512 here):
        # len(top) * 2u * sqrt(K) of max|dY|, doubled as the bound
        kmax = max(i for i, _ in dims)
        tol = 4 * len(top) * 2.0 ** -11 * kmax ** 0.5
        assert abs(s / B - L) <= 1e-3 * abs(L)
        upd = np.abs(newp - p0.double().numpy()).max()
        assert np.abs(got_p - newp).max() <= tol * upd + 1e-7
        assert np.abs(got_dy - dYr).max() <= tol * np.abs(dYr).max()
