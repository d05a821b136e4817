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


# ---------------------------------------------------------------- NEXT-4: richer replay statistics
def trace_report(arrival_us: np.ndarray, end_us: np.ndarray, trace_off: np.ndarray) -> dict:
    """Per trace (paper tables P:1557-1578 / P:1633-1653):
    max and nearest-rank p95 of the response end - r (µs), makespan = last end -
    first arrival (µs), completions (every task completes: O7 has no horizon),
    and throughput = completions per minute of makespan."""
    nt = len(trace_off) - 1
    out = {"max_resp_us": np.zeros(nt, np.int64), "p95_resp_us": np.zeros(nt, np.int64),
           "makespan_us": np.zeros(nt, np.int64), "n": np.zeros(nt, np.int64)}
    for t in range(nt):
        lo, hi = int(trace_off[t]), int(trace_off[t + 1])
        if hi == lo:
            continue
        resp = np.sort(np.asarray(end_us[lo:hi], np.int64) - np.asarray(arrival_us[lo:hi], np.int64))
        out["max_resp_us"][t] = resp[-1]
        out["p95_resp_us"][t] = resp[max(0, math.ceil(0.95 * len(resp)) - 1)]
        out["makespan_us"][t] = int(np.max(end_us[lo:hi])) - int(np.min(arrival_us[lo:hi]))
        out["n"][t] = hi - lo
    return out


def throughput_per_min(n: int, makespan_us: int) -> float:
    """completions / (makespan in minutes)."""
    return 0.0 if makespan_us <= 0 else n / (makespan_us / 60e6)


def utilization(util, makespan_us, cores) -> tuple[np.ndarray, np.ndarray]:
    """Executor utilization (the simulated analogue of the paper's
    "CPU / GPU util." overhead table): busy time / makespan per executor, from
    the replay's busy accumulators (`simulate(..., want_util=True)`).  The CPU
    fraction divides by cores x makespan (every core is an executor); a trace
    with no makespan or no cores reports 0."""
    ms = np.asarray(makespan_us, np.float64)
    c = np.broadcast_to(np.asarray(cores, np.float64), ms.shape)
    g = np.where(ms > 0, util["gpu_busy_us"] / np.where(ms > 0, ms, 1.0), 0.0)
    den = ms * c
    cp = np.where(den > 0, util["cpu_busy_us"] / np.where(den > 0, den, 1.0), 0.0)
    return g, cp
