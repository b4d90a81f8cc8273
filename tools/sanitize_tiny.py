"""The tiny-config hot path under compute-sanitizer: profile ->
threshold -> classify -> group -> training loop (graph, fused and two-kernel
steps) -> standalone fwd / bwd+SGD -> scatter / cold packing.  Small sizes so
every tool finishes; usage:
  compute-sanitizer --tool memcheck python tools/sanitize_tiny.py"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2103_00686_b200 as m  # noqa: E402
from paper_2103_00686_b200.pipeline import FaePipeline  # noqa: E402

dev = torch.device("cuda", 0)
for fused in ("1", "0"):
    os.environ["FAE_FUSED"] = fused
    for name in ("tiny", "ali", "tb64"):
        if name == "tb64" and fused == "1":
            continue
        if name == "tiny":
            cfg = gen.CONFIGS["tiny"]
            R, t, small = 6_000, 1e-2, 0
        elif name == "tb64":   # D = 64: medium segments packed per CTA, staged-id forward at 2 CTAs / SM
            cfg = gen.Config("tb64", [max(3, r // 20_000) for r in gen.TERABYTE_ROWS], 64, 256, 1, records=3_000)
            R, t, small = 3_000, 1e-6, 1 << 40
        else:
            cfg = gen.Config("ali-s", [500, 2000, 90], 16, 32, 0, 3, 12, records=2_000)
            R, t, small = 2_000, 1e-3, 0
        ds = gen.make_dataset(cfg, n_records=R, seed=3).to(dev)
        pipe = FaePipeline(cfg.rows, cfg.dim, cfg.batch, cfg.pool, max_pool=max(cfg.pool_hi, 1))
        prep = pipe.preprocess(ds.idx, ds.off, R, x_pct=5.0, seed=7, t=t, small_table_bytes=small)
        W = gen.make_weights(sum(cfg.rows), cfg.dim, device=dev)
        W_hot = pipe.extract(W, prep).clone()
        pipe.group(prep)
        nb = min(prep.packed["n_hot_batches"], 6)
        S = cfg.batch * cfg.n_tables
        dY = gen.make_dy(nb * S, cfg.dim, device=dev).view(nb, S, cfg.dim)
        Y = torch.zeros(S, cfg.dim, device=dev)
        pipe.train(W_hot, 0, nb, dY, Y, 0.05)
        for i in range(min(2, nb)):
            idx, off, n_bags = pipe.batch_args(prep, i)
            pipe.step(W_hot, prep, i, Y[:n_bags], dY[i, :n_bags], 0.05)
        m.fae_scatter_hot(pipe.ctx, W_hot, W)
        nc = prep.packed["n_cold"]
        cold_idx = torch.empty(max(ds.n_lookups, 1), dtype=torch.int32, device=dev)
        cold_off = torch.empty(nc * cfg.n_tables + 1, dtype=torch.int64, device=dev) if ds.off is not None else None
        m.fae_pack_cold(pipe.ctx, cfg.rows, cfg.dim, ds.idx, cfg.pool, R, prep.cold_ids, nc, cold_idx,
                        off=ds.off, cold_off=cold_off)
        pipe.ctx.check()
        torch.cuda.synchronize()
        print(f"{name} fused={fused}: ok, launches={pipe.ctx.launches}", flush=True)
# round 2: the mixed epoch (cold grouping in global ids, scratch release), the
# DLRM hot step and a scheduled FAE epoch (cuBLAS GEMMs + interaction / loss
# kernels + the grouped loop), and the exchange loop on a 1-rank communicator
import numpy as np  # noqa: E402
from paper_2103_00686_b200.pipeline import FaeTrainer, MixedEpoch  # noqa: E402

os.environ["FAE_FUSED"] = "1"
cfg = gen.CONFIGS["tiny"]
R = 3_000
ds = gen.make_dataset(cfg, n_records=R, seed=5).to(dev)
pipe = FaePipeline(cfg.rows, cfg.dim, cfg.batch, cfg.pool)
prep = pipe.preprocess(ds.idx, None, R, x_pct=5.0, seed=3, t=1e-2, small_table_bytes=0)
W = gen.make_weights(sum(cfg.rows), cfg.dim, device=dev)
W_hot = pipe.extract(W, prep).clone()
ep = MixedEpoch(pipe, prep, W, ds.idx, None, R, W_hot)
Tn, D = cfg.n_tables, cfg.dim
dims = gen.dlrm_dims(4, [12, D], [20, 1], Tn, D)
params = gen.dlrm_pad(gen.make_dlrm_params(dims, device=dev), dims)
tds = gen.make_dataset(cfg, n_records=256, seed=5, record_base=R)
base = torch.tensor(np.concatenate([[0], np.cumsum(cfg.rows)])[:Tn], device=dev)
tidx = (tds.idx.to(dev).view(256, Tn) + base).view(-1).to(torch.int32)
tr = FaeTrainer(ep, 4, [12, D], [20, 1], params, gen.make_dense(R, 4, device=dev), gen.make_labels(R, 4, device=dev),
                tidx, None, 256, gen.make_dense(256, 4, device=dev, record_base=R),
                gen.make_labels(256, 4, device=dev, record_base=R), tf32=True)
sched = m.Scheduler(ep.n_cold_batches, ep.n_hot_batches, 50.0)
tr.run_epoch(sched, 0.05, 0.01)
ep.finish()
pipe.ctx.check()
ep.cold.ctx.check()
torch.cuda.synchronize()
print(f"trainer epoch: ok, swaps={sched.swaps}", flush=True)
if os.environ.get("SANITIZE_NCCL") == "1":
    os.environ["FAE_FORCE_MERGE"] = "1"
    p2 = FaePipeline(cfg.rows, cfg.dim, cfg.batch, cfg.pool)
    m.fae_comm_init(p2.ctx, m.fae_get_nccl_id(), 0, 1)
    pr2 = p2.preprocess(ds.idx, None, R, x_pct=5.0, seed=3, t=1e-2, small_table_bytes=0)
    Wh2 = p2.extract(W, pr2).clone()
    p2.group(pr2)
    nb = pr2.packed["n_hot_batches"]
    S = cfg.batch * Tn
    dY = gen.make_dy(nb * S, D, device=dev).view(nb, S, D)
    p2.train(Wh2, 0, nb, dY, torch.zeros(S, D, device=dev), 0.05)
    p2.ctx.check()
    torch.cuda.synchronize()
    print("exchange loop: ok", flush=True)
print("sanitize_tiny done")
