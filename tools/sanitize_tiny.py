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
    for name in ("tiny", "ali"):
        if name == "tiny":
            cfg = gen.CONFIGS["tiny"]
            R, t, small = 6_000, 1e-2, 0
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
print("sanitize_tiny done")
