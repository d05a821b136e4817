"""NEXT-2 oracle: offline profiling primitives — TEST INFRASTRUCTURE ONLY.

Only tests/ (and bench.py's cpu legs) may import this module.

* fit_weighted_rule: the weighted rule "assign a weight to each category by
  learning a linear regression" as SPEC S:181-189 fixes it:
  ordinary least squares of the target on the six rule scores plus an
  intercept, by the normal equations with ridge damping 1e-8 on the diagonal
  (S:184); DegenerateDesign when the damped normal matrix is numerically
  singular (condition estimate > 1e12).  fp64; np.linalg.solve is the
  linear-algebra step.
* quantile_threshold: Eq. 4 "tau = quantile_k" as the nearest-rank
  quantile of S:208-216: sort ascending, return the element at ceil(k n) - 1.
* u_max: the maximum prediction over the training set.
"""
from __future__ import annotations

import math

import numpy as np

RIDGE = 1e-8
COND_MAX = 1e12


class DegenerateDesign(ValueError):
    pass


def design_matrix(feat: np.ndarray) -> np.ndarray:
    """[1, S, Y, M, V, O, P] per record (the six rule scores)."""
    f = np.asarray(feat)[:, :6].astype(np.float64)
    return np.hstack([np.ones((f.shape[0], 1)), f])


def fit_weighted_rule(feat: np.ndarray, target: np.ndarray) -> np.ndarray:
    """Returns (c, w_S, w_Y, w_M, w_V, w_O, w_P) minimising ||X b - y||^2 + 1e-8 ||b||^2."""
    x = design_matrix(feat)
    y = np.asarray(target, np.float64)
    if x.shape[0] < 7:
        raise DegenerateDesign("fewer than 7 records (S:183)")
    if not x[:, 1:].any():
        raise DegenerateDesign("feature matrix is all zero (S:183)")
    a = x.T @ x + RIDGE * np.eye(7)
    if np.linalg.cond(a) > COND_MAX:
        raise DegenerateDesign("damped normal matrix is numerically singular")
    return np.linalg.solve(a, x.T @ y)


def quantile_threshold(scores: np.ndarray, k: float) -> float:
    s = np.sort(np.asarray(scores, np.float64))
    if len(s) == 0:
        raise ValueError("EmptyScores (S:212)")
    return float(s[max(0, math.ceil(k * len(s)) - 1)])


def u_max(scores: np.ndarray) -> float:
    return float(np.max(np.asarray(scores, np.float64)))
