"""Uniform-over-hot-set control: the training kernels on hot
batches whose hot ids are uniform over a hot table far larger than L2
(>= 9 GB), so no Zipf head stays cached: the honest HBM gather roofline of
the step.  The hot CSR is synthesised directly (26 tables, disjoint hot-id
ranges, single-lookup bags); profile/classify are not part of this control.

usage: python tools/uniform_control.py [--dim 16|64] [--batches 200]
prints one JSON line per dim."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
import paper_2103_00686_b200 as fae  # noqa: E402
from paper_2103_00686_b200.pipeline import FaePipeline, Prepared  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def run(dim, nb, batch, Tn=26):
    dev = torch.device("cuda", 0)
    H = (9 << 30) // (dim * 4) // Tn * Tn          # >= 9 GB hot table
    per = H // Tn
    rows = [per] * Tn
    pipe = FaePipeline(rows, dim, batch, 1)
    n_hot = nb * batch
    g = torch.Generator(device=dev).manual_seed(20260101 + dim)
    hot_idx = torch.randint(0, per, (n_hot, Tn), device=dev, dtype=torch.int32, generator=g)
    hot_idx += (torch.arange(Tn, device=dev, dtype=torch.int32) * per).view(1, Tn)
    hot_idx = hot_idx.view(-1).contiguous()
    prep = Prepared(counts=None, T=[], n_sampled=0, thresh={"H_total": H}, hot_ids=None, cold_ids=None,
                    hot_idx=hot_idx, hot_off=None,
                    packed={"n_hot": n_hot, "n_hot_lookups": n_hot * Tn, "n_hot_batches": nb})
    W_hot = torch.empty(H, dim, device=dev).uniform_(-0.05, 0.05, generator=g)
    S = batch * Tn
    n_dy = max(1, (256 << 20) // (S * dim * 4))
    dY = torch.empty(n_dy, S, dim, device=dev).uniform_(-1, 1, generator=g)
    Y = torch.empty(S, dim, device=dev)
    pipe.group(prep)
    gi = fae.fae_group_info(pipe.ctx)
    fae.fae_set_kernel_timing(pipe.ctx, 1)
    pipe.train(W_hot, 0, nb, dY, Y, 0.01)          # warm-up (graph capture)
    torch.cuda.synchronize()
    fae.fae_set_kernel_timing(pipe.ctx, 1)
    pipe.train(W_hot, 0, nb, dY, Y, 0.01)
    torch.cuda.synchronize()
    pipe.ctx.check()
    kt = fae.fae_get_kernel_timing(pipe.ctx)
    L = S                                           # single-lookup bags
    U = gi["segments"] / nb
    F = gi["free_segments"] / nb
    red = 4 * L + 32 * U + 4 * dim * L + 8 * dim * U
    fwd = 4 * L + 4 * dim * L + 4 * dim * S
    if kt["fused"]:
        us = kt["reduce"][0] / max(kt["reduce"][1], 1) * 1e3
        b = red + 4 * L + 4 * dim * S + (16 + 4 * dim) * F
        kern = "k_grp_fused_pdl"
        parts = {"fused_us": us}
    else:
        fus = kt["fwd"][0] / max(kt["fwd"][1], 1) * 1e3
        rus = kt["reduce"][0] / max(kt["reduce"][1], 1) * 1e3
        us, b, kern = rus, red, "k_grp_reduce_pdl"
        parts = {"fwd_us": fus, "reduce_us": rus, "fwd_frac": fwd / (fus * 1e-6) / 1e9 / peak()}
    achieved = b / (us * 1e-6) / 1e9
    print(json.dumps({"control": "uniform hot ids", "dim": dim, "hot_rows": H, "hot_table_gb": H * dim * 4 / 1e9,
                      "batch": batch, "batches": nb, "distinct_rows_per_batch": U, "kernel": kern,
                      "us_per_launch": us, "bytes_per_launch": b, "achieved_gbs": achieved,
                      "peak_gbs": peak(), "frac": achieved / peak(), **parts}), flush=True)
    del W_hot, dY, pipe
    torch.cuda.empty_cache()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=0)
    ap.add_argument("--batches", type=int, default=200)
    a = ap.parse_args()
    for d, B in ([(a.dim, 2048 if a.dim == 16 else 4096)] if a.dim else [(16, 2048), (64, 4096)]):
        run(d, a.batches, B)
