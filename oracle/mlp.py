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
