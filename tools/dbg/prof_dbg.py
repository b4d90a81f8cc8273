import sys, os, threading
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
os.environ["FAE_LOOPBACK"] = "1"
import numpy as np, torch
import gen, oracle
import paper_2103_00686_b200 as m
from paper_2103_00686_b200.pipeline import FaePipeline

def run(world, cfgname, R, x, seed=4242, conc=True):
    cfg = gen.CONFIGS[cfgname]
    full = gen.make_dataset(cfg, n_records=R, seed=17)
    samp_ref = oracle.sample(R, x, seed)
    counts_ref, T_ref, st = oracle.histogram(full.rows, full.idx, full.off, full.fixed_pool, R, samp_ref)
    per = -(-R // world)
    bounds = [(min(r * per, R), min((r + 1) * per, R)) for r in range(world)]
    dev = torch.device("cuda", 0)
    out = [None]*world
    def body(rank):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            lo, hi = bounds[rank]
            ds = gen.make_dataset(cfg, n_records=hi - lo, seed=17, device=dev, record_base=lo)
            pipe = FaePipeline(cfg.rows, cfg.dim, cfg.batch, cfg.pool, max_world=max(world,1))
            pipe.ctx.set_stream(s)
            if world > 1:
                m.fae_comm_init_loopback(pipe.ctx, 77 + world*1000 + int(x), rank, world)
            counts = torch.empty(sum(cfg.rows), dtype=torch.int32, device=dev)
            samp = torch.empty(max(hi - lo, 1), dtype=torch.int64, device=dev)
            T, ns = m.fae_profile(pipe.ctx, cfg.rows, cfg.dim, ds.idx, ds.off, ds.fixed_pool, hi - lo, x,
                                  seed, counts, samp, record_base=lo, n_records_global=R)
            s.synchronize()
            out[rank] = (samp[:ns].cpu().numpy() + lo, counts.cpu().numpy().view(np.uint32), T)
    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    [t.start() for t in ts]; [t.join() for t in ts]
    ids = np.concatenate([o[0] for o in out])
    print(f"world={world} {cfgname} R={R} x={x}: ids_ok={np.array_equal(ids, samp_ref)}", end=" ")
    c = out[0][1]
    bad = np.nonzero(c != counts_ref)[0]
    rb = np.concatenate([[0], np.cumsum(cfg.rows)])
    print(f"bad={len(bad)} T_ok={list(out[0][2])==list(T_ref)}")
    if len(bad):
        z = np.searchsorted(rb, bad, side="right") - 1
        print("  bad tables:", np.unique(z, return_counts=True))
        print("  first:", bad[:5], c[bad[:5]], counts_ref[bad[:5]])
        print("  sum gpu", c.sum(dtype=np.int64), "ref", counts_ref.sum(dtype=np.int64))

run(1, "kaggle", 200_000, 100.0)
run(1, "kaggle", 50_000, 100.0)
run(4, "kaggle", 200_000, 100.0)
run(4, "kaggle", 200_000, 5.0)
run(1, "kaggle", 200_000, 5.0)
