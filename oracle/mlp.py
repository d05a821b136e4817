"""NEXT-1 oracle: the lightweight MLP m_theta — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py may import this module;
the product package never does.

The paper's Eq. 1 regressor u_J = m_theta(RuleGen(J)) is a
"data-driven black-box lightweight (LW) multi-layer perceptron ... that takes
the six rule-based scores as features" with "four layers of
hidden size [100, 200, 200, 100]" (v2 P:1547).  SPEC S:160-165 fixes
the layer dims [6, 100, 200, 200, 100, 1], rectifier on hidden layers,
identity on the output, and S:192 clamps the output below at 0.  Plain fp64
numpy, layer by layer, in that order.  Weights are row-major [out][in].
"""
from __future__ import annotations

import numpy as np

DIMS = (6, 100, 200, 200, 100, 1)


def mlp_predict(feat: np.ndarray, weights, biases) -> np.ndarray:
    """u = max(0, W5 relu(W4 relu(W3 relu(W2 relu(W1 x + b1) + b2) + b3) + b4) + b5),
    x = the six rule scores {S, Y, M, V, O, P} (feat columns 0..5)."""
    x = np.asarray(feat)[:, :6].astype(np.float64)
    for layer, (w, b) in enumerate(zip(weights, biases)):
        x = x @ np.asarray(w, np.float64).T + np.asarray(b, np.float64)
        if layer < len(DIMS) - 2:
            x = np.maximum(x, 0.0)  # rectifier on hidden layers
    return np.maximum(x[:, 0], 0.0)  # clamp below at 0


def mlp_abs_pass(feat: np.ndarray, weights, biases) -> np.ndarray:
    """The same pass on |W|, |b|, |x| with no rectifier: an upper bound on the
    magnitude of every partial sum of the output, used to state the tolerance of
    reduced-precision evaluations (DESIGN.md §7 K7)."""
    x = np.abs(np.asarray(feat)[:, :6].astype(np.float64))
    for w, b in zip(weights, biases):
        x = x @ np.abs(np.asarray(w, np.float64)).T + np.abs(np.asarray(b, np.float64))
    return x[:, 0]


# ---------------------------------------------------------------- NEXT-2 (optional part): training
# Alg. 1 offline part, "Minimize L_MSE <- ||m_theta(r_J) - l_J||^2" (v2
# P:1384), "train the model with a learning rate of 1e-4" "for 100
# epochs"; mini-batch gradient descent with the Adam
# update rule (beta1 0.9, beta2 0.999, eps 1e-8) on the mean-squared error.
# Readings (DESIGN.md R-TRAIN): the loss is taken on the raw output (the clamp
# at 0 of S:192 belongs to inference); batch k of epoch e is the requests
# pi_e(i), i in [k*B, min(n, (k+1)*B)), with the affine permutation
# pi_e(i) = (a_e * i + b_e) mod n of epoch_perm(); one Adam step per batch,
# t counting steps over all epochs; the epoch loss is the sum of the squared
# errors seen in the epoch's forward passes divided by n.

BETA1, BETA2, ADAM_EPS = 0.9, 0.999, 1e-8


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def epoch_perm(n: int, seed: int, epoch: int):
    """(a, b) of epoch `epoch`'s permutation i -> (a*i + b) mod n: h = splitmix64(seed
    + epoch); a = 1 + h mod n, incremented until gcd(a, n) = 1; b = (h >> 32) mod n."""
    from math import gcd
    h = _splitmix64((seed + epoch) & 0xFFFFFFFFFFFFFFFF)
    a = 1 + h % n
    while gcd(a, n) != 1:
        a += 1
    return a % n, (h >> 32) % n


def mlp_forward_raw(x: np.ndarray, weights, biases):
    """Activations of every layer for inputs x [B, 6] (fp64): returns the list
    [x, h1, h2, h3, h4, z] with ReLU on the hidden layers, z the raw output [B]."""
    acts = [x]
    for layer, (w, b) in enumerate(zip(weights, biases)):
        y = acts[-1] @ w.T + b
        if layer < len(DIMS) - 2:
            y = np.maximum(y, 0.0)
        acts.append(y)
    acts[-1] = acts[-1][:, 0]
    return acts


def mlp_grads(x: np.ndarray, y: np.ndarray, weights, biases):
    """Loss mean((z - y)^2) over the batch and its gradients with respect to
    every weight and bias (backpropagation through the ReLUs; the derivative of
    ReLU at 0 is taken as 0)."""
    acts = mlp_forward_raw(x, weights, biases)
    z = acts[-1]
    bsz = x.shape[0]
    loss = float(np.mean((z - y) ** 2))
    dz = (2.0 / bsz) * (z - y)[:, None]  # [B, 1]
    gw, gb = [None] * 5, [None] * 5
    for layer in range(4, -1, -1):
        a_in = acts[layer]
        gw[layer] = dz.T @ a_in
        gb[layer] = dz.sum(axis=0)
        if layer > 0:
            da = dz @ weights[layer]
            dz = da * (acts[layer] > 0.0)
    return loss, gw, gb


def mlp_train_adam(feat: np.ndarray, y: np.ndarray, weights, biases, epochs: int, batch: int, lr: float,
                   seed: int):
    """Trains in fp64 from the given weights; returns (weights, biases, epoch losses)."""
    ws = [np.asarray(w, np.float64).copy() for w in weights]
    bs = [np.asarray(b, np.float64).copy() for b in biases]
    mw = [np.zeros_like(w) for w in ws]
    vw = [np.zeros_like(w) for w in ws]
    mb = [np.zeros_like(b) for b in bs]
    vb = [np.zeros_like(b) for b in bs]
    x_all = np.asarray(feat)[:, :6].astype(np.float64)
    y_all = np.asarray(y, np.float64)
    n = x_all.shape[0]
    t = 0
    losses = []
    for e in range(epochs):
        a, b = epoch_perm(n, seed, e)
        order = (a * np.arange(n, dtype=np.int64) + b) % n if n > 1 else np.zeros(1, np.int64)
        sq = 0.0
        for k in range(0, n, batch):
            idx = order[k:k + batch]
            loss, gw, gb = mlp_grads(x_all[idx], y_all[idx], ws, bs)
            sq += loss * len(idx)
            t += 1
            c1, c2 = 1.0 / (1.0 - BETA1 ** t), 1.0 / (1.0 - BETA2 ** t)
            for p, g, m, v in list(zip(ws, gw, mw, vw)) + list(zip(bs, gb, mb, vb)):
                m *= BETA1
                m += (1.0 - BETA1) * g
                v *= BETA2
                v += (1.0 - BETA2) * g * g
                p -= lr * (m * c1) / (np.sqrt(v * c2) + ADAM_EPS)
        losses.append(sq / n)
    return ws, bs, np.asarray(losses)
