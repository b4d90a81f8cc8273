"""World-size-2 tests of the multi-GPU host logic on CPU (gloo).

The data-path exchanges run in NCCL inside libfae on GPUs; here the same
protocols are checked with the oracle as the compute: (1) rank shards of the
generated dataset are exactly the slices of the unsharded one; (2) the
sparse hot-gradient exchange — every rank all-gathers the (row, G) lists and
merges them in rank order — yields bit-identical replicas equal to the
single-process update of the concatenated batch;
(3) the batch-count agreement and id broadcast helpers of dist.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_00686_b200 import dist as fdist
        out = {}
        # (3) helpers
        out["max"] = fdist.max_over_ranks(10 + 5 * rank)
        out["sum"] = fdist.sum_over_ranks(1.5 * (rank + 1))
        payload = bytes(range(128)) if rank == 0 else None
        out["bcast"] = fdist.broadcast_bytes(payload, 0, 128)
        # (1) sharded generation
        cfg = gen.Config("ali-small", [300, 700, 50], 16, 64, 0, 20, 100, records=200)
        base, n = fdist.shard(100, rank)
        mine = gen.make_dataset(cfg, n_records=n, record_base=base, seed=9)
        full = gen.make_dataset(cfg, n_records=200, seed=9)
        lo, hi = int(full.off[base * 3]), int(full.off[(base + n) * 3])
        out["shard_ok"] = bool(torch.equal(full.idx[lo:hi], mine.idx)) and \
            bool(torch.equal(full.off[base * 3:(base + n) * 3 + 1] - lo, mine.off))
        # (2) sparse gradient exchange, rank-ordered merge, SGD
        H, D, B, lr = 500, 8, 64, 0.05
        rng = np.random.default_rng(123)
        idx_all = (rng.zipf(1.3, B * world) % H).astype(np.int32)
        dY_all = rng.uniform(-1, 1, (B * world, D)).astype(np.float32)
        W0 = rng.uniform(-0.05, 0.05, (H, D)).astype(np.float32)
        sl = slice(rank * B, (rank + 1) * B)
        rows, G = oracle.emb_grad(H, D, idx_all[sl], None, 1, B, dY_all[sl])
        gathered = [None] * world
        dist.all_gather_object(gathered, (rows.tolist(), G.astype(np.float32).tolist()))
        acc = {}
        for rr, gg in gathered:            # rank order, then ascending row
            for r, g in zip(rr, gg):
                acc.setdefault(r, np.zeros(D, np.float64))
                acc[r] += np.asarray(g, np.float64)
        W = W0.copy()
        for r in sorted(acc):
            W[r] = (W[r].astype(np.float64) - np.float64(np.float32(lr)) * acc[r]).astype(np.float32)
        out["W"] = W
        ref, _ = oracle.emb_bwd_sgd(W0, idx_all, None, 1, B * world, dY_all, lr)
        out["ref"] = ref
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_helpers(results):
    assert results[0]["max"] == results[1]["max"] == 15
    assert results[0]["sum"] == results[1]["sum"] == 4.5
    assert results[0]["bcast"] == results[1]["bcast"] == bytes(range(128))


def test_shards_are_slices_of_the_global_dataset(results):
    assert results[0]["shard_ok"] and results[1]["shard_ok"]


def test_sparse_gradient_exchange(results):
    W0, W1 = results[0]["W"], results[1]["W"]
    assert np.array_equal(W0, W1)                  # replicas bit-identical
    ref = results[0]["ref"]
    assert np.all(np.abs(W0 - ref) <= 1e-6 + 1e-5 * np.abs(ref))
