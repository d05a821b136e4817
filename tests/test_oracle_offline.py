"""Pins of the NEXT-2 offline-profiling oracle (oracle/offline.py) from SPEC
S:185-187 and S:214-216 and the mathematics of least squares."""
import numpy as np
import pytest

from oracle.offline import DegenerateDesign, fit_weighted_rule, quantile_threshold, u_max


def _feat(n, seed):
    rng = np.random.default_rng(seed)
    f = np.zeros((n, 8), np.uint16)
    f[:, :6] = rng.integers(0, 30, (n, 6))
    return f


def test_exact_linear_targets_are_recovered():
    # S:185 "targets exactly 2*vague + 5 with other features zero -> (0,0,0,2,0,0), intercept 5, within 1e-6"
    f = _feat(500, 1)
    y = 2.0 * f[:, 3] + 5.0
    b = fit_weighted_rule(f, y)
    assert np.allclose(b, [5, 0, 0, 0, 2, 0, 0], atol=1e-6)
    # any exact linear map is recovered
    w = np.array([6.0, 2.0, 1.5, 4.0, 3.0, 5.0, 5.0])
    y = f[:, :6] @ w[1:] + w[0]
    assert np.allclose(fit_weighted_rule(f, y), w, atol=1e-6)


def test_constant_target_gives_the_intercept():
    # S:186 "constant target c with nonconstant features -> intercept c, coefficients 0 within 1e-6"
    f = _feat(400, 2)
    b = fit_weighted_rule(f, np.full(400, 7.25))
    assert abs(b[0] - 7.25) < 1e-6 and np.abs(b[1:]).max() < 1e-6


def test_residual_is_optimal():
    # S:187 residual <= that of the zero-coefficient model; and the normal-equation residual
    # is orthogonal to the design columns (first-order optimality), up to the ridge term
    f = _feat(1000, 3)
    rng = np.random.default_rng(4)
    y = rng.normal(20, 5, 1000)
    b = fit_weighted_rule(f, y)
    x = np.hstack([np.ones((1000, 1)), f[:, :6].astype(np.float64)])
    r = y - x @ b
    assert r @ r <= y @ y
    assert np.abs(x.T @ r - 1e-8 * b).max() < 1e-6 * np.abs(x.T @ y).max()
    for j in range(7):  # any single perturbation of a coefficient increases the residual
        for d in (-1e-3, 1e-3):
            bb = b.copy()
            bb[j] += d
            rr = y - x @ bb
            assert rr @ rr >= r @ r


def test_degenerate_design():
    with pytest.raises(DegenerateDesign):
        fit_weighted_rule(np.zeros((100, 8), np.uint16), np.arange(100.0))
    with pytest.raises(DegenerateDesign):
        fit_weighted_rule(_feat(5, 1), np.arange(5.0))


def test_nearest_rank_quantile():
    # S:214-215
    assert quantile_threshold(np.arange(1, 11), 0.9) == 9
    assert quantile_threshold([5.0], 0.3) == 5.0
    s = np.random.default_rng(5).random(1000)
    for k in (0.001, 0.1, 0.5, 0.9, 0.999, 1.0):
        assert quantile_threshold(s, k) == np.sort(s)[int(np.ceil(k * 1000)) - 1]
    assert quantile_threshold(s, 1.0) == u_max(s)
    # monotone in k
    ks = np.linspace(0.01, 1, 50)
    q = [quantile_threshold(s, k) for k in ks]
    assert all(a <= b for a, b in zip(q, q[1:]))


def test_trace_report_pins():
    from oracle.offline import throughput_per_min, trace_report
    # responses {1,2,3} -> max 3; single task -> max = p95; p95 vs sort oracle
    r = np.array([0, 0, 0, 5], np.int64)
    e = np.array([1, 2, 3, 9], np.int64)
    rep = trace_report(r, e, np.array([0, 3, 4]))
    assert rep["max_resp_us"].tolist() == [3, 4] and rep["p95_resp_us"].tolist() == [3, 4]
    assert rep["makespan_us"].tolist() == [3, 4] and rep["n"].tolist() == [3, 1]
    rng = np.random.default_rng(1)
    resp = rng.integers(0, 10**9, 10**4)
    rep = trace_report(np.zeros(10**4, np.int64), resp, np.array([0, 10**4]))
    assert rep["p95_resp_us"][0] == np.sort(resp)[9499]
    # 60 tasks in 2 minutes -> 30/min; zero completions -> 0
    assert throughput_per_min(60, 120_000_000) == 30.0 and throughput_per_min(0, 0) == 0.0


def _small_traces(offload=True, consolidate=True):
    """Config-3-shaped traces (4 LMs, Poisson ramp) scored by the oracle."""
    import oracle
    from rtgen import configs
    lex = oracle.Lexicon(configs.read_lexicon())
    d = configs.traces(3, range(7), 300, lambda t: t % 4)
    for p in d["profiles"]:
        p["offload"] = int(offload)
        p["consolidate"] = int(consolidate)
    n = len(d["arrival_us"])
    f = oracle.rule_gen(lex, d["data"], d["offsets"])
    u = np.zeros(n, np.float32)
    k = np.zeros(n, np.uint64)
    D = np.zeros(n, np.uint32)
    for t in range(len(d["trace_off"]) - 1):
        lo, hi = int(d["trace_off"][t]), int(d["trace_off"][t + 1])
        p = d["profiles"][int(d["trace_prof"][t])]
        u[lo:hi] = oracle.predict(f[lo:hi], d["regressors"][int(d["trace_prof"][t])])
        k[lo:hi], D[lo:hi] = oracle.key(u[lo:hi], f[lo:hi], p, r_us=d["arrival_us"][lo:hi])
    st, end, ut = oracle.simulate(d["arrival_us"], d["true_len"], u, k, D, d["trace_off"], d["profiles"],
                                  d["trace_prof"], want_end=True, want_util=True)
    return d, k, end, ut


def test_utilization_pins_special_cases():
    # S:405 "single serial batch occupying the whole makespan -> GPU fraction 1.0";
    # S:406 "no CPU offloads -> CPU fraction 0.0"
    import oracle
    from oracle.offline import trace_report, utilization
    from rtgen import configs
    p = dict(configs.paper_lms()[0], offload=0, consolidate=1, policy=oracle.POLICY["UP"])
    r = np.zeros(1, np.int64)
    ln = np.array([40], np.uint16)
    st, end, ut = oracle.simulate(r, ln, np.ones(1, np.float32), np.zeros(1, np.uint64), np.full(1, 10**9, np.uint32),
                                  np.array([0, 1]), p, want_end=True, want_util=True)
    dur = p["setup_us"] + p["base_us"] + p["eta_us"] * 40      # S:386-391 batch latency
    assert end[0] == dur and ut["gpu_busy_us"][0] == dur and ut["gpu_batches"][0] == 1
    rep = trace_report(r, end, np.array([0, 1]))
    g, c = utilization(ut, rep["makespan_us"], p["cores"])
    assert g[0] == 1.0 and c[0] == 0.0
    d, k, end, ut = _small_traces(offload=False)
    assert (ut["cpu_busy_us"] == 0).all() and (ut["cpu_tasks"] == 0).all()


def test_utilization_matches_interval_union():
    # S:407 "random workload -> fractions match an independent interval-union oracle":
    # rebuild every executor interval from the per-task end times alone (a GPU
    # batch = the GPU-class tasks sharing one end time, duration setup + base +
    # eta * max len; a CPU task runs gamma * (base + eta * len) before its end),
    # merge them, and compare with the event loop's accumulators.
    from oracle.offline import trace_report, utilization
    d, k, end, ut = _small_traces()
    rep = trace_report(d["arrival_us"], end, d["trace_off"])
    for t in range(len(d["trace_off"]) - 1):
        lo, hi = int(d["trace_off"][t]), int(d["trace_off"][t + 1])
        p = d["profiles"][int(d["trace_prof"][t])]
        cls = (k[lo:hi] >> np.uint64(63)).astype(bool)
        ln = d["true_len"][lo:hi].astype(np.int64)
        e = end[lo:hi]
        gpu = {}
        for i in np.nonzero(~cls)[0]:
            gpu.setdefault(int(e[i]), []).append(i)
        iv = sorted((ee - (p["setup_us"] + p["base_us"] + p["eta_us"] * int(ln[b].max())), ee) for ee, b in gpu.items())
        for (s0, e0), (s1, e1) in zip(iv, iv[1:]):
            assert e0 <= s1                       # one GPU: batches never overlap
        assert all(len(b) <= p["C"] for b in gpu.values())
        union = sum(e1 - s0 for s0, e1 in iv)
        assert ut["gpu_busy_us"][t] == union and ut["gpu_batches"][t] == len(gpu)
        cpu = np.nonzero(cls)[0]
        assert ut["cpu_tasks"][t] == len(cpu)
        cdur = p["gamma"] * (p["base_us"] + p["eta_us"] * ln[cpu])
        assert ut["cpu_busy_us"][t] == int(cdur.sum())
        # per-core intervals do not overlap: at most `cores` CPU tasks at once
        ev = sorted([(int(e[i] - c), 1) for i, c in zip(cpu, cdur)] + [(int(e[i]), -1) for i in cpu],
                    key=lambda x: (x[0], x[1]))
        live = 0
        for _, dl in ev:
            live += dl
            assert live <= p["cores"]
    g, c = utilization(ut, rep["makespan_us"], [d["profiles"][int(x)]["cores"] for x in d["trace_prof"]])
    assert ((0 <= g) & (g <= 1)).all() and ((0 <= c) & (c <= 1)).all()
    assert (ut["cpu_tasks"] > 0).any() and (ut["gpu_batches"] > 0).all()
