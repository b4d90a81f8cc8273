import os, sys, subprocess
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, gen
import paper_2103_00686_b200 as m
from paper_2103_00686_b200.pipeline import FaePipeline
name, first_mode, nb, R = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
cfg = gen.CONFIGS[name]
dev = torch.device("cuda", 0)
ds = gen.make_dataset(cfg, n_records=R, device=dev)
pipe = FaePipeline(cfg.rows, cfg.dim, cfg.batch, cfg.pool, max_pool=max(cfg.pool_hi, 1))
mode = m.BUDGET_EXACT if cfg.budget_bytes else m.FIXED_T
prep = pipe.preprocess(ds.idx, ds.off, R, x_pct=5.0, seed=1, mode=mode, t=cfg.t, budget_bytes=cfg.budget_bytes, small_table_bytes=cfg.small_bytes)
W = gen.make_weights(sum(cfg.rows), cfg.dim, device=dev)
W_hot = pipe.extract(W, prep)
pipe.group(prep)
nbt = prep.packed["n_hot_batches"]
first = {"zero": 0, "mid": nbt // 2, "end": nbt - nb}[first_mode]
S = cfg.batch * cfg.n_tables
dY = gen.make_dy(nb * S, cfg.dim, seed=77, device=dev).view(nb, S, cfg.dim)
Y = torch.zeros(S, cfg.dim, device=dev)
pipe.train(W_hot, first, nb, dY, Y, 0.01)
try:
    pipe.ctx.check(); print(name, first_mode, nb, R, "nbt", nbt, "fused", os.environ.get("FAE_FUSED"), "OK", flush=True)
except Exception as e:
    print(name, first_mode, nb, R, "nbt", nbt, "fused", os.environ.get("FAE_FUSED"), "FAIL", e, flush=True)
