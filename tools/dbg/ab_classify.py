"""A/B: fae_classify legacy vs bulk kernel on a full-size workload."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, gen
import paper_2103_00686_b200 as m
from paper_2103_00686_b200.pipeline import FaePipeline
name = sys.argv[1]
cfg = gen.CONFIGS[name]
R = cfg.records
dev = torch.device("cuda", 0)
ds = gen.make_dataset(cfg, n_records=R, device=dev)
res = {}
for legacy in ("1", "0"):
    os.environ["FAE_CLS_LEGACY"] = legacy
    pipe = FaePipeline(cfg.rows, cfg.dim, cfg.batch, cfg.pool, max_pool=max(cfg.pool_hi, 1))
    mode = m.BUDGET_EXACT if cfg.budget_bytes else m.FIXED_T
    prep = pipe.preprocess(ds.idx, ds.off, R, x_pct=5.0, seed=1, mode=mode, t=cfg.t, budget_bytes=cfg.budget_bytes, small_table_bytes=cfg.small_bytes)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        pk = m.fae_classify(pipe.ctx, cfg.rows, cfg.dim, ds.idx, ds.off, cfg.pool, R, cfg.batch, prep.hot_ids, prep.cold_ids, prep.hot_idx, prep.hot_off)
        ts.append((time.perf_counter() - t0) * 1e3)
    res[legacy] = (sorted(ts)[2], pk["n_hot"], prep.hot_ids[:pk["n_hot"]].clone(), prep.hot_idx[:pk["n_hot_lookups"]].clone())
    del pipe, prep
print(name, "legacy %.2f ms  bulk %.2f ms" % (res["1"][0], res["0"][0]), "same:", res["1"][1] == res["0"][1] and torch.equal(res["1"][2], res["0"][2]) and torch.equal(res["1"][3], res["0"][3]))
