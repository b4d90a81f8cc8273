"""CPU ORACLE of the DLRM hot step — TEST INFRASTRUCTURE ONLY.

Only tests/ (and bench.py's oracle legs) may import this module; the product
path never does, and nothing here comes from it.  Plain numpy in float64,
written from the model the paper trains (§5 `tab:benchmarks`,
P:L516-526: DLRM, bottom MLP over the dense features, the embedding bags of
the sparse features, "dot" feature interaction, top MLP, logarithmic loss
P:L559-560; SGD P:L230), definitions in the order they are stated:

  bottom:   h_0 = dense;  h_{l+1} = relu(h_l W_l^T + b_l)          (all layers)
  interact: T = [h_bot, Y_0, ..., Y_{Tn-1}]  (F = Tn + 1 vectors of D)
            Z_ij = <T_i, T_j> for i > j, in (i, j) row-major order
            x_top = [h_bot, Z]                        (D + F(F-1)/2 values)
  top:      g_0 = x_top;  g_{l+1} = relu(g_l V_l^T + c_l), the last layer
            linear: z = g V^T + c (one logit per sample)
  loss:     mean over the batch of  -(y log s(z) + (1-y) log(1 - s(z)))
  backward: the chain rule of the above (written out below, no autograd);
            dY (the embedding bags' gradient, input of a9) = dT_1..Tn
  SGD:      every MLP weight / bias  p -= lr * dL/dp   (R13)

DLRM's ReLU on every bottom layer and a linear last top layer (sigmoid in
the loss) are the published DLRM defaults (external to PAPER.md, which only
names the layer widths) — DESIGN.md R32.  A matmul is a library primitive
step (numpy @ in float64).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def layer_dims(n_dense: int, bottom: List[int], top: List[int], n_tables: int, D: int):
    """[(in, out)] of every bottom then top layer; bottom[-1] must equal D."""
    assert bottom[-1] == D
    dims, prev = [], n_dense
    for w in bottom:
        dims.append((prev, w))
        prev = w
    F = n_tables + 1
    prev = D + F * (F - 1) // 2
    for w in top:
        dims.append((prev, w))
        prev = w
    assert top[-1] == 1
    return dims


def unpack(params: np.ndarray, dims) -> List[Tuple[np.ndarray, np.ndarray]]:
    """Flat parameter layout (include/fae.h fae_dlrm): per layer W [out][in]
    row-major then b [out], bottom layers first."""
    out, o = [], 0
    for i, n in dims:
        W = params[o:o + n * i].reshape(n, i)
        o += n * i
        b = params[o:o + n]
        o += n
        out.append((W, b))
    assert o == params.size
    return out


def tril_pairs(F: int):
    return [(i, j) for i in range(1, F) for j in range(i)]


def forward(params, dims, n_bottom, dense, Y, label):
    """Returns (mean loss, cache).  dense [B][n_dense], Y [B][Tn][D]."""
    p = unpack(np.asarray(params, np.float64), dims)
    B = dense.shape[0]
    h = [np.asarray(dense, np.float64)]
    for l in range(n_bottom):
        W, b = p[l]
        h.append(np.maximum(h[-1] @ W.T + b, 0.0))
    Yd = np.asarray(Y, np.float64)
    T = np.concatenate([h[-1][:, None, :], Yd], axis=1)          # [B][F][D]
    F = T.shape[1]
    pairs = tril_pairs(F)
    Z = np.empty((B, len(pairs)))
    for k, (i, j) in enumerate(pairs):
        Z[:, k] = np.sum(T[:, i, :] * T[:, j, :], axis=1)
    g = [np.concatenate([h[-1], Z], axis=1)]
    nl = len(dims)
    for l in range(n_bottom, nl):
        W, b = p[l]
        a = g[-1] @ W.T + b
        g.append(a if l == nl - 1 else np.maximum(a, 0.0))
    z = g[-1][:, 0]
    y = np.asarray(label, np.float64)
    # -(y log s + (1-y) log(1-s)) = max(z,0) - z y + log(1 + exp(-|z|))
    loss = np.maximum(z, 0.0) - z * y + np.log1p(np.exp(-np.abs(z)))
    return float(loss.mean()), dict(p=p, h=h, T=T, pairs=pairs, g=g, z=z, y=y, B=B)


def backward_sgd(params, dims, n_bottom, cache, lr):
    """(updated params, dY [B][Tn][D], gradient of every parameter)."""
    p, h, T, pairs, g, z, y, B = (cache[k] for k in ("p", "h", "T", "pairs", "g", "z", "y", "B"))
    nl = len(dims)
    grads = [None] * nl
    s = 1.0 / (1.0 + np.exp(-z))
    d = ((s - y) / B)[:, None]                                    # dL/dz
    for l in range(nl - 1, n_bottom - 1, -1):
        W, b = p[l]
        x = g[l - n_bottom]
        grads[l] = (d.T @ x, d.sum(axis=0))
        d = d @ W
        if l > n_bottom:                                          # relu of the layer below
            d = d * (x > 0.0)
    D = T.shape[2]
    dT = np.zeros_like(T)
    dT[:, 0, :] += d[:, :D]
    dZ = d[:, D:]
    for k, (i, j) in enumerate(pairs):
        dT[:, i, :] += dZ[:, k:k + 1] * T[:, j, :]
        dT[:, j, :] += dZ[:, k:k + 1] * T[:, i, :]
    d = dT[:, 0, :] * (h[-1] > 0.0)
    for l in range(n_bottom - 1, -1, -1):
        W, b = p[l]
        x = h[l]
        grads[l] = (d.T @ x, d.sum(axis=0))
        d = d @ W
        if l > 0:
            d = d * (x > 0.0)
    flat = []
    for (W, b), (gW, gb) in zip(p, grads):
        flat.append((W - lr * gW).reshape(-1))
        flat.append(b - lr * gb)
    return np.concatenate(flat), dT[:, 1:, :], grads
