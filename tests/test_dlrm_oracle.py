"""Pins of the DLRM oracle (oracle/dlrm.py, NEXT-2) — CPU only: a
hand-derived one-sample fixture (golden), the symmetric zero-weight case
(loss = ln 2), saturation, and central finite differences of the loss for
every parameter and every embedding-bag value (the analytic backward), plus
lr = 0 and the SGD identity p' = p - lr g."""
import math
import os

import numpy as np

from oracle import dlrm

GOLD = os.path.join(os.path.dirname(__file__), "golden", "dlrm_tiny.txt")


def _fixture():
    ln = [l for l in open(GOLD) if l.strip() and not l.startswith("#")]
    parts = [p.strip() for p in ln[0].split("|")]
    vals = [np.array([float(v) for v in p.split(",")]) for p in parts]
    dldz = float(ln[1].split()[1])
    return vals, dldz


def test_hand_derived_forward_and_loss_gradient():
    (params, dense, Y, label, loss), dldz = _fixture()
    dims = dlrm.layer_dims(1, [2], [1], 1, 2)
    L, cache = dlrm.forward(params, dims, 1, dense.reshape(1, 1), Y.reshape(1, 1, 2), label)
    assert abs(L - loss[0]) < 1e-15
    _, _, grads = dlrm.backward_sgd(params, dims, 1, cache, 0.0)
    assert abs(grads[-1][1][0] - dldz) < 1e-15          # dL/dc = s(z) - y


def _rand_model(rng, n_dense=5, bottom=(7, 4), top=(9, 6, 1), Tn=3, D=4, B=6):
    dims = dlrm.layer_dims(n_dense, list(bottom), list(top), Tn, D)
    n = sum(i * o + o for i, o in dims)
    params = rng.normal(0, 0.4, n)
    dense = rng.normal(0, 1, (B, n_dense))
    Y = rng.normal(0, 0.5, (B, Tn, D))
    label = (rng.random(B) < 0.5).astype(np.float64)
    return dims, len(bottom), params, dense, Y, label


def test_zero_weights_give_ln2():
    rng = np.random.default_rng(1)
    dims, nb, params, dense, Y, label = _rand_model(rng)
    L, _ = dlrm.forward(np.zeros_like(params), dims, nb, dense, np.zeros_like(Y), label)
    assert abs(L - math.log(2.0)) < 1e-15


def test_saturation():
    dims = dlrm.layer_dims(1, [2], [1], 1, 2)
    params = np.array([1, 2, 0, -1, 0, 0, 0, 40.0])      # z = 40
    L, _ = dlrm.forward(params, dims, 1, np.ones((1, 1)), np.zeros((1, 1, 2)), np.ones(1))
    assert 0 <= L < 1e-17
    L0, _ = dlrm.forward(params, dims, 1, np.ones((1, 1)), np.zeros((1, 1, 2)), np.zeros(1))
    assert abs(L0 - 40.0) < 1e-12


def test_finite_differences():
    rng = np.random.default_rng(7)
    dims, nb, params, dense, Y, label = _rand_model(rng)
    L, cache = dlrm.forward(params, dims, nb, dense, Y, label)
    lr = 0.1
    newp, dY, grads = dlrm.backward_sgd(params, dims, nb, cache, lr)
    flat_g = np.concatenate([np.concatenate([gW.reshape(-1), gb]) for gW, gb in grads])
    assert np.allclose(newp, params - lr * flat_g, rtol=0, atol=1e-15)
    eps = 1e-6
    for k in rng.choice(params.size, 60, replace=False):
        pp, pm = params.copy(), params.copy()
        pp[k] += eps
        pm[k] -= eps
        fd = (dlrm.forward(pp, dims, nb, dense, Y, label)[0] - dlrm.forward(pm, dims, nb, dense, Y, label)[0]) / (2 * eps)
        assert abs(fd - flat_g[k]) <= 1e-7 + 1e-5 * abs(fd), (k, fd, flat_g[k])
    for idx in [(0, 0, 0), (1, 2, 3), (5, 1, 2), (3, 0, 1)]:
        Yp, Ym = Y.copy(), Y.copy()
        Yp[idx] += eps
        Ym[idx] -= eps
        fd = (dlrm.forward(params, dims, nb, dense, Yp, label)[0] - dlrm.forward(params, dims, nb, dense, Ym, label)[0]) / (2 * eps)
        assert abs(fd - dY[idx]) <= 1e-7 + 1e-5 * abs(fd)


def test_lr_zero_identity():
    rng = np.random.default_rng(3)
    dims, nb, params, dense, Y, label = _rand_model(rng)
    _, cache = dlrm.forward(params, dims, nb, dense, Y, label)
    newp, _, _ = dlrm.backward_sgd(params, dims, nb, cache, 0.0)
    assert np.array_equal(newp, params)
