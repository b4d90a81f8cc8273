import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, gen
import paper_2103_00686_b200 as m
from paper_2103_00686_b200.pipeline import FaePipeline
name = sys.argv[1]
cfg = gen.CONFIGS[name]; R = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.records
dev = torch.device("cuda", 0)
ds = gen.make_dataset(cfg, n_records=R, device=dev)
pipe = FaePipeline(cfg.rows, cfg.dim, cfg.batch, cfg.pool, max_pool=max(cfg.pool_hi, 1))
mode = m.BUDGET_EXACT if cfg.budget_bytes else m.FIXED_T
prep = pipe.preprocess(ds.idx, ds.off, R, x_pct=5.0, seed=1, mode=mode, t=cfg.t, budget_bytes=cfg.budget_bytes, small_table_bytes=cfg.small_bytes)
torch.cuda.synchronize()
