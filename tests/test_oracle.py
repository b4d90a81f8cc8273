"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something OTHER than itself: values the
paper prints (tests/golden/*, cited), closed forms, textbook/library routines
(numpy bincount / add.at, torch sparse mm and embedding_bag autograd in fp64,
scipy's Student-t), brute force on tiny inputs, and invariants the method
implies.  A plausible mistake (dropped term, wrong sign or index, transposed
operand, > vs >=, wrong rounding) fails at least one of them.
"""
import math
import os

import numpy as np
import pytest
import torch

import gen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ----------------------------------------------------------------------------
# Eq. 1 worked example
# ----------------------------------------------------------------------------
def test_eq1_worked_example():
    for t, T, x, H, kmin, hot, cold in _golden("eq1_worked_example.txt"):
        Hc = oracle.cutoff(float(t), int(T), float(x))
        assert Hc == float(H)
        assert oracle.kmin_from_cutoff(Hc) == int(kmin)
        # one large table with two rows: k = 303 is hot, k = 302 is cold
        counts = np.array([int(hot), int(cold)], np.uint32)
        km = oracle.kmin_fixed_t([2], 1 << 20, 0, [int(T)], float(t), float(x))
        assert km[0] == int(kmin)
        tags = oracle.tag_rows([2], 1 << 20, 0, counts, km)
        assert tags.tolist() == [1, 0]


def test_cutoff_x100_and_tiny_cutoff():
    # x = 100 -> H = t*T; t*T = 1, x = 50 -> 0.5 -> one access needed
    assert oracle.cutoff(1e-3, 1000, 100.0) == 1.0
    assert oracle.cutoff(1e-3, 1000, 50.0) == 0.5
    assert oracle.kmin_from_cutoff(0.5) == 1
    assert oracle.kmin_from_cutoff(1.0) == 1
    assert oracle.kmin_from_cutoff(1.0000001) == 2
    assert oracle.kmin_from_cutoff(0.0) == 1   # R25 clamp


# ----------------------------------------------------------------------------
# O1 sampler
# ----------------------------------------------------------------------------
def test_sample_identity_and_counts():
    R = 1000
    assert oracle.sample(R, 100.0, 7).tolist() == list(range(R))
    assert oracle.lib().or_sample_count(60_500_000, 5.0) == 3_025_000
    assert oracle.lib().or_sample_count(10_000, 5.0) == 500
    assert oracle.lib().or_sample_count(10, 0.0) == -1
    assert oracle.lib().or_sample_count(10, 100.5) == -1
    assert len(oracle.sample(19, 5.0, 1)) == 0   # floor(0.95) = 0


def test_sample_selection_property():
    R, x, seed = 5000, 5.0, 123
    ids = oracle.sample(R, x, seed)
    assert len(ids) == 250
    assert np.all(np.diff(ids) > 0)          # ascending, distinct
    keys = np.array([oracle.key(seed, i) for i in range(R)], dtype=np.uint64)
    chosen = np.zeros(R, bool)
    chosen[ids] = True
    # every chosen key is below every unchosen key (the k smallest)
    assert keys[chosen].max() < keys[~chosen].min()


def test_sample_inclusion_frequency():
    # uniform without replacement: each record included w.p. ~ x/100
    R, x, n_seeds = 200, 5.0, 400
    hits = np.zeros(R)
    for s in range(n_seeds):
        hits[oracle.sample(R, x, 1000 + s)] += 1
    freq = hits / n_seeds
    sd = math.sqrt(0.05 * 0.95 / n_seeds)
    assert abs(freq.mean() - 0.05) < 1e-12       # exactly k per draw
    assert np.mean(np.abs(freq - 0.05) < 4 * sd) > 0.99


def test_key_is_splitmix64():
    # the documented counter hash (R6): splitmix64 of seed + (i+1)*golden
    def mix(z):
        M = (1 << 64) - 1
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 & M
        z = (z ^ (z >> 27)) * 0x94D049BB133111EB & M
        return z ^ (z >> 31)
    # published splitmix64 first outputs for state 0 (Vigna's reference):
    assert mix(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF
    assert oracle.key(0, 0) == 0xE220A8397B1DCDAF
    for s, i in [(0, 5), (99, 0), (2**63, 12345)]:
        assert oracle.key(s, i) == mix((s + (i + 1) * 0x9E3779B97F4A7C15) & ((1 << 64) - 1))


# ----------------------------------------------------------------------------
# O2 embedding logger
# ----------------------------------------------------------------------------
def test_histogram_spec_examples():
    # three records each accessing row 7 of table 0 once -> k[7] = 3
    counts, T, st = oracle.histogram([10], [7, 7, 7], None, 1, 3, [0, 1, 2])
    assert st == 0 and counts[7] == 3 and counts.sum() == 3 and T[0] == 3
    # multi-hot record {2, 2, 5} -> k[2] = 2, k[5] = 1
    counts, T, st = oracle.histogram([10], [2, 2, 5], [0, 3], 0, 1, [0])
    assert counts[2] == 2 and counts[5] == 1 and counts.sum() == 3


def test_histogram_brute_force_tiny():
    cfg = gen.CONFIGS["tiny"]
    ds = gen.make_dataset(cfg, n_records=2000)
    samp = oracle.sample(ds.n_records, 5.0, 9)
    counts, T, st = oracle.histogram(ds.rows, ds.idx, None, 1, ds.n_records,
                                     samp)
    assert st == 0
    idx = ds.idx.numpy().reshape(ds.n_records, 4)
    for z in range(4):
        bc = np.bincount(idx[samp, z], minlength=1000)
        assert np.array_equal(counts[z * 1000:(z + 1) * 1000], bc)
        assert T[z] == ds.n_records
        assert counts[z * 1000:(z + 1) * 1000].sum() == len(samp)


def test_histogram_variable_pooling_and_range_error():
    cfg = gen.CONFIGS["alibaba"]
    small = gen.Config("ali-small", [300, 700, 50], 16, 64, 0, 20, 100,
                       records=300)
    ds = gen.make_dataset(small)
    samp = np.arange(0, 300, 3)
    counts, T, st = oracle.histogram(ds.rows, ds.idx, ds.off, 0, 300, samp)
    assert st == 0
    off = ds.off.numpy(); idx = ds.idx.numpy()
    base = np.concatenate([[0], np.cumsum(ds.rows)])
    ref = np.zeros(base[-1], np.int64)
    Tref = np.zeros(3, np.int64)
    for r in range(300):
        for z in range(3):
            b = r * 3 + z
            Tref[z] += off[b + 1] - off[b]
            if r % 3 == 0:
                np.add.at(ref, base[z] + idx[off[b]:off[b + 1]], 1)
    assert np.array_equal(counts, ref) and np.array_equal(T, Tref)
    assert cfg.pool == 0
    _, _, st = oracle.histogram([4], [1, 9], None, 1, 2, [0, 1])
    assert st == oracle.INDEX_RANGE


# ----------------------------------------------------------------------------
# a3 threshold (Eq. 1 / BUDGET_EXACT / small-table rule)
# ----------------------------------------------------------------------------
def _tiny_counts(seed=3, R=4000):
    cfg = gen.CONFIGS["tiny"]
    ds = gen.make_dataset(cfg, n_records=R, seed=seed)
    samp = oracle.sample(R, 5.0, seed)
    counts, T, _ = oracle.histogram(ds.rows, ds.idx, None, 1, R, samp)
    return ds, counts, T


def test_fixed_t_brute_force_and_monotone():
    ds, counts, T = _tiny_counts()
    prev = None
    for t in [1e-3, 3e-3, 1e-2, 3e-2]:   # x = 5, T = 4000 -> kmin 1, 1, 2, 6
        km = oracle.kmin_fixed_t(ds.rows, 16, 0, T, t, 5.0)
        H = t * 4000 * 5 / 100
        assert all(k == max(1, math.ceil(H)) for k in km)
        hot = oracle.tag_rows(ds.rows, 16, 0, counts, km)
        assert np.array_equal(hot, (counts >= km[0]).astype(np.uint8))
        if prev is not None:                 # t1 < t2 => hot(t1) ⊇ hot(t2)
            assert np.all(prev >= hot)
        prev = hot


def test_small_table_rule():
    # tables < 1 MB are hot in full; rows*dim*4 = 2^20 is large
    rows = [100, (1 << 20) // 64]
    counts = np.zeros(sum(rows), np.uint32)
    km = oracle.kmin_fixed_t(rows, 16, 1 << 20, [10, 10], 0.5, 5.0)
    hot = oracle.tag_rows(rows, 16, 1 << 20, counts, km)
    assert hot[:100].all() and not hot[100:].any()
    assert km[0] == 0 and km[1] == 1


def test_budget_exact_feasible_maximal_monotone():
    ds, counts, T = _tiny_counts()
    Tref = int(T.max())
    prevK = None
    for budget in [64 * 50, 64 * 200, 64 * 800, 64 * 2000, 64 * 4000]:
        r = oracle.budget_exact(ds.rows, 16, 0, counts, T, 5.0, budget)
        assert r["status"] == 0
        K = r["K"]
        km = r["kmin"]
        # all T equal -> K_z = K
        assert all(k == K for k in km)
        b = oracle.hot_bytes(ds.rows, 16, 0, counts, km)
        bruteb = int((counts >= K).sum()) * 64
        assert b == bruteb <= budget                        # feasible
        if K > 1:                                           # maximal
            assert int((counts >= K - 1).sum()) * 64 > budget
        else:
            assert r["slack"] == 1
        assert r["t_final"] == K / (Tref * 5.0 / 100.0)
        if prevK is not None:
            assert K <= prevK                               # monotone in L
        prevK = K


def test_budget_linear_scan_agrees():
    # bisection == plain linear scan over K (the definition "smallest K")
    ds, counts, T = _tiny_counts(seed=11)
    for budget in [640, 6400, 25600]:
        r = oracle.budget_exact(ds.rows, 16, 0, counts, T, 5.0, budget)
        K = 1
        while int((counts >= K).sum()) * 64 > budget:
            K += 1
        assert r["K"] == K


def test_budget_unequal_T_and_infeasible():
    rows = [2000, 2000, 10]
    counts = np.zeros(4010, np.uint32)
    rng = np.random.default_rng(0)
    counts[:4000] = rng.integers(0, 50, 4000)
    T = np.array([1000, 400, 5])
    small = 64 * 10 + 1            # third table small (640 B < 641 B)
    r = oracle.budget_exact(rows, 16, small, counts, T, 5.0, 64 * 300 + 640)
    K = r["K"]
    assert r["kmin"][0] == K and r["kmin"][1] == max(1, math.ceil(K * 400 / 1000))
    assert r["kmin"][2] == 0
    b = oracle.hot_bytes(rows, 16, small, counts, r["kmin"])
    assert b <= 64 * 300 + 640
    r2 = oracle.budget_exact(rows, 16, small, counts, T, 5.0, 100)
    assert r2["status"] == oracle.BUDGET_INFEASIBLE
    # uniform degenerate case: equal counts, budget = all rows -> K=1
    cu = np.full(1000, 7, np.uint32)
    r3 = oracle.budget_exact([1000], 16, 0, cu, [1000], 5.0, 64 * 1000)
    assert r3["K"] == 1 and r3["slack"] == 1
    r4 = oracle.budget_exact([1000], 16, 0, cu, [1000], 5.0, 64 * 999)
    assert r4["K"] == 8  # nothing fits until the cutoff passes the common count


# ----------------------------------------------------------------------------
# Eqs. 2-4 estimate
# ----------------------------------------------------------------------------
def test_t_quantile_readings():
    from scipy import stats
    for p, df, val, tol in _golden("t_quantile.txt"):
        assert abs(stats.t.ppf(float(p), int(df)) - float(val)) <= float(tol)


def test_estimate_degenerate_cases():
    k = np.full(64 * 1024, 9, np.uint32)
    e = oracle.estimate(k, 5, n=35, m=1024, chunk_seed=1)
    assert e["s"] == 0.0 and e["ybar"] == 1024 and e["est"] == len(k)
    assert e["lo"] == e["hi"] == len(k)
    e = oracle.estimate(k, 10)      # cutoff above max -> 0
    assert e["ybar"] == 0 and e["est"] == 0 and e["hi"] == 0
    k2 = np.arange(20 * 1024, dtype=np.uint32) % 7   # N = 20 < n = 35: exact
    e = oracle.estimate(k2, 3)
    assert e["exact"] and e["est"] == int((k2 >= 3).sum())


def test_estimate_matches_textbook_formula():
    rng = np.random.default_rng(5)
    Nz = 300 * 1024 + 77
    k = rng.integers(0, 10, Nz).astype(np.uint32)
    e = oracle.estimate(k, 7, n=35, m=1024, chunk_seed=42, t_q=3.6007)
    ch = e["chunks"]
    assert len(set(ch.tolist())) == 35 and ch.min() >= 0 and ch.max() < 300
    assert np.all(np.diff(ch) > 0)
    C = np.array([(k[c * 1024:(c + 1) * 1024] >= 7).sum() for c in ch])
    assert np.array_equal(C, e["C"])
    ybar = C.mean()
    s = C.std(ddof=1)
    hw = 3.6007 * math.sqrt((300 - 35) / 300 * s * s / 35)
    assert abs(e["ybar"] - ybar) < 1e-9
    assert abs(e["s"] - s) < 1e-9
    sc = Nz / 1024
    assert abs(e["lo"] - (ybar - hw) * sc) < 1e-6
    assert abs(e["hi"] - (ybar + hw) * sc) < 1e-6
    # chunk choice = the 35 smallest keys
    keys = np.array([oracle.key(42, c) for c in range(300)], np.uint64)
    assert set(ch.tolist()) == set(np.argsort(keys, kind="stable")[:35].tolist())


def test_estimate_within_10pct_on_zipf():
    # P:L455, L462 ("within 10% of the actual values", 99.9% CI): the exact
    # count lies inside [lo, hi] and the point estimate is within 10% for
    # >= 95% of 20 seeds on a Zipf(1.1) logger (uniform-looking after the
    # Feistel scatter), at a cutoff that makes ~30% of rows hot.
    n = 400_000
    u = gen.uniform01(77, torch.arange(2_000_000))
    cdf = gen.zipf_cdf(n, 1.1, "cpu")
    rank = torch.searchsorted(cdf, u).clamp(max=n - 1)
    rows = gen.feistel(rank, n, 5)
    k = np.bincount(rows.numpy(), minlength=n).astype(np.uint32)
    kmin = 2
    exact = int((k >= kmin).sum())
    ok = cover = 0
    for s in range(20):
        e = oracle.estimate(k, kmin, chunk_seed=s)
        ok += abs(e["est"] - exact) <= 0.1 * exact
        cover += e["lo"] <= exact <= e["hi"]
    assert ok >= 19 and cover >= 19


# ----------------------------------------------------------------------------
# O4 remap, O5 classify, O6 pack, O7 extract
# ----------------------------------------------------------------------------
def test_remap_bijection_and_rank():
    rows = [5, 3, 4]
    hot = np.array([1, 0, 1, 1, 0, 0, 0, 1, 1, 1, 0, 1], np.uint8)
    rm, base, H = oracle.remap(rows, hot)
    assert H == hot.sum() == 7
    assert rm.tolist() == [0, -1, 1, 2, -1, -1, -1, 3, 4, 5, -1, 6]
    assert base.tolist() == [0, 3, 4, 7]
    assert sorted(rm[rm >= 0].tolist()) == list(range(H))


def test_classify_brute_force_and_rules():
    ds, counts, T = _tiny_counts(seed=4)
    km = oracle.kmin_fixed_t(ds.rows, 16, 0, T, 3e-3, 5.0)
    hot = oracle.tag_rows(ds.rows, 16, 0, counts, km)
    rm, base, H = oracle.remap(ds.rows, hot)
    flag = oracle.classify(ds.rows, ds.idx, None, 1, ds.n_records, rm)
    idx = ds.idx.numpy().reshape(-1, 4) + np.arange(4) * 1000
    brute = hot[idx].all(axis=1)
    assert np.array_equal(flag.astype(bool), brute)
    # one cold index in one table poisons the record
    rows = [4, 4]
    hotv = np.array([1, 1, 1, 1, 1, 0, 1, 1], np.uint8)
    rm2, _, _ = oracle.remap(rows, hotv)
    f = oracle.classify(rows, [0, 0, 3, 1, 2, 3], None, 1, 3, rm2)
    assert f.tolist() == [1, 0, 1]
    # empty bag: vacuously hot (R19)
    f = oracle.classify([4], [], [0, 0], 0, 1, np.zeros(4, np.int32))
    assert f.tolist() == [1]


def test_pack_spec_example_and_invariants():
    for flags, B, hb, cb in _golden("pack_example.txt"):
        flag = np.array([int(v) for v in flags.split(",")], np.uint8)
        B = int(B)
        rows = [10]
        idx = np.arange(10, dtype=np.int32)
        rm = np.where(flag == 1, np.cumsum(flag) - 1, -1).astype(np.int32)
        p = oracle.pack(rows, idx, None, 1, 10, rm, flag)
        sizes = lambda n: [min(B, n - i) for i in range(0, n, B)]
        assert sizes(p["n_hot"]) == [int(v) for v in hb.split(",")]
        assert sizes(p["n_cold"]) == [int(v) for v in cb.split(",")]
    ds, counts, T = _tiny_counts(seed=8)
    km = oracle.kmin_fixed_t(ds.rows, 16, 0, T, 3e-3, 5.0)
    hot = oracle.tag_rows(ds.rows, 16, 0, counts, km)
    rm, base, H = oracle.remap(ds.rows, hot)
    flag = oracle.classify(ds.rows, ds.idx, None, 1, ds.n_records, rm)
    p = oracle.pack(ds.rows, ds.idx, None, 1, ds.n_records, rm, flag)
    allids = np.concatenate([p["hot_ids"], p["cold_ids"]])
    assert np.array_equal(np.sort(allids), np.arange(ds.n_records))  # partition
    assert np.all(np.diff(p["hot_ids"]) > 0) and np.all(np.diff(p["cold_ids"]) > 0)
    hi = p["hot_idx"]
    assert hi.min() >= 0 and hi.max() < H                            # purity
    cold_lookups = 4 * p["n_cold"]
    assert p["n_hot_lookups"] + cold_lookups == T.sum()              # conservation
    gidx = ds.idx.numpy().reshape(-1, 4)[p["hot_ids"]] + np.arange(4) * 1000
    assert np.array_equal(hi.reshape(-1, 4), rm[gidx])


def test_pack_variable_pooling():
    small = gen.Config("ali-small", [300, 700, 50], 16, 64, 0, 20, 100,
                       records=200)
    ds = gen.make_dataset(small, seed=4)
    rng = np.random.default_rng(1)
    hot = (rng.random(1050) < 0.97).astype(np.uint8)
    rm, base, H = oracle.remap(ds.rows, hot)
    flag = oracle.classify(ds.rows, ds.idx, ds.off, 0, 200, rm)
    p = oracle.pack(ds.rows, ds.idx, ds.off, 0, 200, rm, flag)
    off = ds.off.numpy(); idx = ds.idx.numpy()
    rb = np.concatenate([[0], np.cumsum(ds.rows)])
    out, offs = [], [0]
    for r in p["hot_ids"]:
        for z in range(3):
            b = r * 3 + z
            out += rm[rb[z] + idx[off[b]:off[b + 1]]].tolist()
            offs.append(len(out))
    assert p["hot_idx"].tolist() == out and p["hot_off"].tolist() == offs


def test_all_hot_probability_closed_form():
    # naive batching of independent inputs with hot prob p gives
    # all-hot batches w.p. p^B; packing makes every hot batch all-hot.
    for p, B, val, tol in _golden("all_hot_probability.txt"):
        assert abs(float(p) ** int(B) - float(val)) <= float(tol) + 1e-12
    rng = np.random.default_rng(0)
    B, p, nb = 256, 0.99, 4000
    flags = (rng.random(B * nb) < p).astype(np.uint8)
    frac = flags.reshape(nb, B).all(axis=1).mean()
    assert abs(frac - p ** B) < 4 * math.sqrt(p ** B * (1 - p ** B) / nb)
    rm = np.zeros(1, np.int32)
    idx = np.where(flags == 1, 0, 1).astype(np.int32)   # row 1 is cold
    rm = np.array([0, -1], np.int32)
    f = oracle.classify([2], idx, None, 1, len(idx), rm)
    pk = oracle.pack([2], idx, None, 1, len(idx), rm, f)
    assert pk["n_hot"] == flags.sum()
    assert np.all(pk["hot_idx"] == 0)


def test_extract_bit_copy():
    W = gen.make_weights(12, 8)
    hot = np.array([0, 1, 1, 0, 1, 0, 0, 0, 1, 1, 0, 1], np.uint8)
    rm, base, H = oracle.remap([12], hot)
    Wh = oracle.extract(W, rm, H)
    assert np.array_equal(Wh, W.numpy()[hot == 1])


# ----------------------------------------------------------------------------
# O8 / O9 hot step
# ----------------------------------------------------------------------------
def _bags(seed, n_bags=40, H=30, dim=8, var=True):
    rng = np.random.default_rng(seed)
    if var:
        sizes = rng.integers(0, 6, n_bags)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    else:
        off = np.arange(n_bags + 1, dtype=np.int64) * 3
    # Zipf-ish repeats
    idx = (rng.zipf(1.5, off[-1]) % H).astype(np.int32)
    W = rng.uniform(-0.05, 0.05, (H, dim)).astype(np.float32)
    dY = rng.uniform(-1, 1, (n_bags, dim)).astype(np.float32)
    return W, idx, off, dY


def _A(idx, off, H):
    n_bags = len(off) - 1
    A = np.zeros((n_bags, H))
    for b in range(n_bags):
        for p in range(off[b], off[b + 1]):
            A[b, idx[p]] += 1
    return A


def test_fwd_is_sparse_dense_product():
    W, idx, off, _ = _bags(1)
    n_bags = len(off) - 1
    Y, st = oracle.emb_fwd(W, idx, off, 0, n_bags)
    assert st == 0
    bag = np.repeat(np.arange(n_bags), np.diff(off))
    Ai = torch.sparse_coo_tensor(
        torch.tensor(np.stack([bag, idx])), torch.ones(len(idx), dtype=torch.float64),
        (n_bags, W.shape[0]))
    ref = torch.sparse.mm(Ai, torch.tensor(W, dtype=torch.float64)).numpy()
    assert np.array_equal(Y, ref.astype(np.float32))
    # empty bags give zero rows
    empty = np.diff(off) == 0
    assert np.all(Y[empty] == 0)
    # single-lookup bag -> bit-exact row (fixed pool 1)
    Y1, _ = oracle.emb_fwd(W, idx[:5], None, 1, 5)
    assert np.array_equal(Y1, W[idx[:5]])


def test_fwd_linearity_and_fixed_pool():
    W, idx, off, _ = _bags(2, var=False)
    n_bags = len(off) - 1
    Ya, _ = oracle.emb_fwd(W, idx, None, 3, n_bags)
    Yb, _ = oracle.emb_fwd(W, idx, off, 0, n_bags)
    assert np.array_equal(Ya, Yb)
    Y2, _ = oracle.emb_fwd(2 * W, idx, None, 3, n_bags)
    assert np.array_equal(Y2, 2 * Ya)    # exact: scaling by 2 is exact in fp


def test_bwd_matches_autograd_and_sgd():
    W, idx, off, dY = _bags(3)
    n_bags = len(off) - 1
    H, dim = W.shape
    lr = 0.01
    Wn, st = oracle.emb_bwd_sgd(W, idx, off, 0, n_bags, dY, lr)
    assert st == 0
    # G = dL/dW for L = sum(Y * dY), Y = embedding_bag(sum) — torch autograd fp64
    Wt = torch.tensor(W, dtype=torch.float64, requires_grad=True)
    Y = torch.nn.functional.embedding_bag(
        torch.tensor(idx, dtype=torch.int64), Wt,
        torch.tensor(off[:-1], dtype=torch.int64), mode="sum",
        include_last_offset=False)
    (Y * torch.tensor(dY, dtype=torch.float64)).sum().backward()
    G = Wt.grad.numpy()
    # G = A^T dY as well (numpy add.at)
    G2 = np.zeros((H, dim))
    bag = np.repeat(np.arange(n_bags), np.diff(off))
    np.add.at(G2, idx, dY[bag].astype(np.float64))
    assert np.allclose(G, G2, rtol=0, atol=1e-12)
    ref = (W.astype(np.float64) - np.float64(np.float32(lr)) * G).astype(np.float32)
    touched = np.zeros(H, bool); touched[idx] = True
    assert np.array_equal(Wn[touched], ref[touched])
    assert np.array_equal(Wn[~touched], W[~touched])        # bit-identical
    W0, _ = oracle.emb_bwd_sgd(W, idx, off, 0, n_bags, dY, 0.0)
    assert np.array_equal(W0, W)                             # lr = 0
    rows, Gs = oracle.emb_grad(H, dim, idx, off, 0, n_bags, dY)
    assert np.array_equal(rows, np.nonzero(touched)[0])
    assert np.allclose(Gs, G[touched], rtol=0, atol=1e-12)


def test_bwd_finite_difference():
    W, idx, off, dY = _bags(4, n_bags=10, H=12, dim=4)
    n_bags = len(off) - 1
    rows, G = oracle.emb_grad(12, 4, idx, off, 0, n_bags, dY)
    W64 = W.astype(np.float64)

    def loss(Wm):
        Y = np.zeros((n_bags, 4))
        for b in range(n_bags):
            for p in range(off[b], off[b + 1]):
                Y[b] += Wm[idx[p]]
        return (Y * dY).sum()
    eps = 1e-6
    for u, r in enumerate(rows[:4]):
        for d in range(4):
            Wp = W64.copy(); Wp[r, d] += eps
            Wm = W64.copy(); Wm[r, d] -= eps
            fd = (loss(Wp) - loss(Wm)) / (2 * eps)
            assert abs(fd - G[u, d]) < 1e-6


def test_sharding_invariance():
    # O10: the sum over G record shards of the per-shard sparse gradients is
    # the gradient of the concatenated batch ("aggregated").
    W, idx, off, dY = _bags(6, n_bags=64, H=40, dim=8, var=False)
    n = 64
    rows_all, G_all = oracle.emb_grad(40, 8, idx, None, 3, n, dY)
    for Gn in (2, 4):
        acc = np.zeros((40, 8))
        per = n // Gn
        for g in range(Gn):
            r, Gg = oracle.emb_grad(40, 8, idx[g * per * 3:(g + 1) * per * 3],
                                    None, 3, per, dY[g * per:(g + 1) * per])
            acc[r] += Gg
        assert np.allclose(acc[rows_all], G_all, rtol=0, atol=1e-12)


# ----------------------------------------------------------------------------
# NEXT-4: CLT-driven statistical optimizer (R27)
# ----------------------------------------------------------------------------
GRID = [10.0 ** (-8 + 0.25 * j) for j in range(29)]


def test_clt_search_uniform_degenerate_slack():
    # every row has the same count and L = bytes of all rows -> the
    # estimate is exact (s = 0, C_i = m), all rows hot at any t below the
    # uniform fraction: the smallest grid t fits (slack), bytes == L
    rows = [40 * 1024]
    cu = np.full(rows[0], 3, np.uint32)
    L = rows[0] * 16 * 4
    r = oracle.clt_search(rows, 16, 1 << 20, cu, [1000], 5.0, L, chunk_seed=9)
    assert r["status"] == 0 and r["slack"] == 1
    assert r["t_final"] == GRID[0] and r["est_bytes"] == L and r["evals"] == 1
    assert list(r["kmin"]) == [1]


def test_clt_search_infeasible():
    # even t = 1e-1 leaves every row hot (all counts above the cutoff): the
    # estimate is N rows > L -> infeasible
    rows = [40 * 1024]
    c = np.full(rows[0], 1000, np.uint32)
    r = oracle.clt_search(rows, 16, 1 << 20, c, [100], 5.0, 1000)
    assert r["status"] == oracle.BUDGET_INFEASIBLE
    # small tables alone above L
    r = oracle.clt_search([100], 16, 1 << 20, np.zeros(100, np.uint32), [10], 5.0, 100)
    assert r["status"] == oracle.BUDGET_INFEASIBLE


def test_clt_search_exact_tables_bisection_bound():
    # tables with fewer than n chunks are scanned exactly (est = exact hot
    # rows), so est_bytes(t) is the exact hot-set size, non-increasing in t.
    # The search then brackets the exact threshold: with t* the smallest t in
    # the final grid cell whose exact bytes fit, t_final - cell/2^8 < t* <=
    # t_final (bisection bound), found here by brute force over a fine scan.
    rng = np.random.default_rng(4)
    rows = [30 * 1024, 20 * 1024]                 # 30, 20 chunks < n = 35
    counts = np.concatenate([rng.zipf(1.3, rows[0]) % 5000,
                             rng.zipf(1.6, rows[1]) % 5000]).astype(np.uint32)
    T = np.array([2_000_000, 500_000])
    for L in [64 * 3000, 64 * 8000, 64 * 20000]:
        r = oracle.clt_search(rows, 16, 1 << 20, counts, T, 5.0, L)
        assert r["status"] == 0 and r["slack"] == 0
        tf = r["t_final"]
        j = min(i for i, g in enumerate(GRID) if g >= tf)
        lo_cell, hi_cell = GRID[j - 1], GRID[j]
        assert lo_cell < tf <= hi_cell
        km = oracle.kmin_fixed_t(rows, 16, 1 << 20, T, tf, 5.0)
        assert list(km) == list(r["kmin"])
        b = oracle.hot_bytes(rows, 16, 1 << 20, counts, km)
        assert b <= L and b == r["est_bytes"]
        d = (hi_cell - lo_cell) / 256
        below = oracle.kmin_fixed_t(rows, 16, 1 << 20, T, tf - d * 1.0001, 5.0)
        assert oracle.hot_bytes(rows, 16, 1 << 20, counts, below) > L or tf - d * 1.0001 <= lo_cell
        # brute force: the exact smallest fitting t in the cell, by a fine scan
        ts = np.linspace(lo_cell, hi_cell, 4097)[1:]
        fit = [t for t in ts
               if oracle.hot_bytes(rows, 16, 1 << 20, counts,
                                   oracle.kmin_fixed_t(rows, 16, 1 << 20, T, t, 5.0)) <= L]
        t_star = min(fit)
        assert tf - d - (ts[1] - ts[0]) <= t_star <= tf


def test_clt_search_budget_on_zipf_estimate():
    # S:L198 [DERIVED]: L = 0.5 x (exact hot bytes at a reference t) on a
    # Zipf(1.05) logger estimated by CLT chunks (N >> n): t_final > t_ref and
    # the exact hot bytes at t_final land in [0.8 L, L] (the Eq. 4 upper bound
    # is what must fit, so the exact set sits just below L; "within
    # 10%").  Reference t with a sizeable hot set (~5% / ~19% of rows).
    n = 400_000
    u = gen.uniform01(78, torch.arange(4_000_000))
    cdf = gen.zipf_cdf(n, 1.05, "cpu")
    rank = torch.searchsorted(cdf, u).clamp(max=n - 1)
    k = np.bincount(gen.feistel(rank, n, 6).numpy(), minlength=n).astype(np.uint32)
    T = [4_000_000 * 20]                      # the sample is x = 5% of T
    for t_ref in (1e-6, 3e-6):
        km = oracle.kmin_fixed_t([n], 16, 1 << 20, T, t_ref, 5.0)
        L = oracle.hot_bytes([n], 16, 1 << 20, k, km) // 2
        ok = 0
        for s in range(10):
            r = oracle.clt_search([n], 16, 1 << 20, k, T, 5.0, L, chunk_seed=100 + s)
            assert r["status"] == 0 and r["t_final"] > t_ref and r["est_bytes"] <= L
            b = oracle.hot_bytes([n], 16, 1 << 20, k, r["kmin"])
            ok += 0.8 * L <= b <= L
        assert ok >= 9


# ----------------------------------------------------------------------------
# NEXT-1: swap sync back to the master tables
# ----------------------------------------------------------------------------
def test_scatter_hot_inverse_of_extract():
    rng = np.random.default_rng(21)
    rows = [300, 500, 200]
    hot = (rng.random(sum(rows)) < 0.3).astype(np.uint8)
    rm, base, H = oracle.remap(rows, hot)
    W = rng.standard_normal((sum(rows), 8)).astype(np.float32)
    # round trip: scattering the extracted table back is the identity
    assert np.array_equal(oracle.scatter_hot(W, oracle.extract(W, rm, H), rm), W)
    # a trained hot table: hot rows take its rows, cold rows stay bit-identical
    W_hot = rng.standard_normal((H, 8)).astype(np.float32)
    W2 = oracle.scatter_hot(W, W_hot, rm)
    g_hot = np.nonzero(rm >= 0)[0]
    assert np.array_equal(W2[g_hot], W_hot[rm[g_hot]])           # brute force
    cold = rm < 0
    assert np.array_equal(W2[cold], W[cold])


# ----------------------------------------------------------------------------
# the all-cores build (cpu_baseline's multi-thread figure) == the serial build
# ----------------------------------------------------------------------------
def test_openmp_build_bit_identical(monkeypatch):
    """oracle.use_omp(True) routes to the same C file compiled with -fopenmp;
    every result must be bit-identical to the serial build (the pragmas split
    independent iterations, integer counts and the backward by row ownership,
    keeping every fp64 sum in its serial order)."""
    monkeypatch.setenv("OMP_NUM_THREADS", "4")
    c = gen.Config("k-small", [max(3, r // 1000) for r in gen.KAGGLE_ROWS], 16, 256, 1, records=20_000)
    ali = gen.Config("a-small", [900, 4000, 90], 8, 64, 0, 5, 40, records=2_000)
    outs = []
    for omp in (False, True):
        oracle.use_omp(omp)
        try:
            res = []
            for cfg, R in ((c, 20_000), (ali, 2_000)):
                ds = gen.make_dataset(cfg, n_records=R, seed=31)
                samp = oracle.sample(R, 5.0, 9)
                counts, T, _ = oracle.histogram(ds.rows, ds.idx, ds.off, ds.fixed_pool, R, samp)
                kmin = oracle.kmin_fixed_t(ds.rows, cfg.dim, 0, T, 1e-4, 5.0)
                hot = oracle.tag_rows(ds.rows, cfg.dim, 0, counts, kmin)
                rm, base, H = oracle.remap(ds.rows, hot)
                flag = oracle.classify(ds.rows, ds.idx, ds.off, ds.fixed_pool, R, rm)
                pk = oracle.pack(ds.rows, ds.idx, ds.off, ds.fixed_pool, R, rm, flag)
                W = gen.make_weights(max(H, 1), cfg.dim).numpy()
                n = min(pk["n_hot"], cfg.batch * 3)
                Tn = ds.n_tables
                if ds.off is None:
                    bi, off, P = pk["hot_idx"][:n * Tn], None, 1
                else:
                    bi, off, P = pk["hot_idx"], pk["hot_off"][:n * Tn + 1], 0
                dY = gen.make_dy(n * Tn, cfg.dim, seed=4).numpy()
                Y, _ = oracle.emb_fwd(W, bi, off, P, n * Tn)
                W2, _ = oracle.emb_bwd_sgd(W, bi, off, P, n * Tn, dY, 0.05)
                res.append((samp, counts, T, flag, pk["hot_idx"], Y, W2))
            outs.append(res)
        finally:
            oracle.use_omp(False)
    for a, b in zip(outs[0], outs[1]):
        for x, y in zip(a, b):
            assert np.array_equal(np.asarray(x), np.asarray(y))
