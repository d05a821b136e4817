"""NEXT-2 parity: rt_fit_rule and rt_quantile against the fp64 oracle
(oracle/offline.py).  The quantile is an order statistic: exact.  The fit's
X^T X is an exact integer sum in fp64 on both sides; X^T y and the solve differ
only in rounding order (Cholesky vs LU), so coefficients agree to ~cond * 1e-16;
the test allows 1e-9 relative to the largest coefficient."""
import math

import numpy as np
import pytest

import oracle
from oracle.offline import fit_weighted_rule, quantile_threshold
from rtgen import configs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2309_06619_b200 as rt  # noqa: E402

DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def ctx():
    return rt.Context(configs.read_lexicon(), 0)


def _dev_feat(f):
    return torch.from_numpy(np.ascontiguousarray(f).view(np.int16)).to(DEV)


@pytest.mark.parametrize("n", [7, 1000, 100003])
def test_fit_on_rule_features(ctx, n):
    d = configs.config2(n=n, gid0=31337)
    f = oracle.rule_gen(oracle.Lexicon(configs.read_lexicon()), d["data"], d["offsets"])
    y = d["true_len"].astype(np.float32)
    if n == 7:  # make the tiny design non-singular
        f[:7, :6] = np.eye(7, 6, dtype=np.uint16) * 3 + 1
    got = ctx.fit_rule(_dev_feat(f), torch.from_numpy(y).to(DEV)).cpu().numpy()
    want = fit_weighted_rule(f, y)
    assert np.abs(got[:7] - want).max() <= 1e-9 * max(1.0, np.abs(want).max())
    assert 0.0 < got[7] <= 1.0


def test_fit_exact_linear(ctx):
    # exactly 2*vague + 5 -> (5, 0, 0, 0, 2, 0, 0)
    rng = np.random.default_rng(8)
    f = np.zeros((5000, 8), np.uint16)
    f[:, :6] = rng.integers(0, 30, (5000, 6))
    y = (2.0 * f[:, 3] + 5.0).astype(np.float32)
    got = ctx.fit_rule(_dev_feat(f), torch.from_numpy(y).to(DEV)).cpu().numpy()
    assert np.allclose(got[:7], [5, 0, 0, 0, 2, 0, 0], atol=1e-6)


@pytest.mark.parametrize("n", [1, 10, 1000, 1 << 20])
def test_quantile_exact(ctx, n):
    rng = np.random.default_rng(n)
    u = rng.gamma(2.0, 10.0, n).astype(np.float32)
    if n >= 1000:
        u[::7] = u[3]  # ties
    du = torch.from_numpy(u).to(DEV)
    for k in (0.001, 0.5, 0.9, 1.0):
        got = ctx.quantile(du, k).cpu().numpy()
        assert got[0] == np.float32(quantile_threshold(u, k)), (n, k)
        assert got[1] == u.max()
    if n == 10:  # 1..10, k = 0.9 -> 9
        got = ctx.quantile(torch.arange(1, 11, dtype=torch.float32, device=DEV), 0.9).cpu().numpy()
        assert got[0] == 9.0 and got[1] == 10.0


def test_offline_errors(ctx):
    with pytest.raises(rt.RtlmError):
        ctx.quantile(torch.zeros(0, dtype=torch.float32, device=DEV), 0.9)
    with pytest.raises(rt.RtlmError):
        ctx.quantile(torch.ones(5, dtype=torch.float32, device=DEV), 0.0)
    with pytest.raises(rt.RtlmError):
        ctx.fit_rule(_dev_feat(np.zeros((6, 8), np.uint16)), torch.zeros(6, dtype=torch.float32, device=DEV))


def test_trace_report_parity(ctx):
    """NEXT-4: per-trace max / p95 / makespan from the replay's end times, exact."""
    from oracle.offline import trace_report
    lex = oracle.Lexicon(configs.read_lexicon())
    d = configs.traces(3, range(100, 112), 1000, lambda t: t % 4)
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
    _, end = oracle.simulate(d["arrival_us"], d["true_len"], u, k, D, d["trace_off"], d["profiles"], d["trace_prof"],
                             want_end=True)
    # ragged traces: sizes 1000, 1, 0, 1024 (rebuild offsets over the same tasks)
    t9 = int(d["trace_off"][9])
    toff = np.concatenate([d["trace_off"][:10], [t9 + 1, t9 + 1, t9 + 1 + 1024]])
    toff = toff.astype(np.uint32)
    arr = torch.from_numpy(d["arrival_us"]).to(DEV)
    e = torch.from_numpy(end).to(DEV)
    rep = ctx.trace_report(arr, e, toff).cpu().numpy()
    want = trace_report(d["arrival_us"], end, toff)
    assert (rep[:, 0] == want["max_resp_us"]).all()
    assert (rep[:, 1] == want["p95_resp_us"]).all()
    assert (rep[:, 2] == want["makespan_us"]).all()
    assert ((rep[:, 3] & 0xFFFFFFFF) == want["n"]).all()


@pytest.mark.gpu
def test_trace_utilization_parity(ctx):
    """NEXT-4: executor busy times from the replay's end times, exact against the
    event loop's own accumulators (oracle.simulate(want_util=True)); offload on
    and off, static and consolidated batching."""
    lex = oracle.Lexicon(configs.read_lexicon())
    for offload, consolidate in ((1, 1), (0, 1), (1, 0)):
        d = configs.traces(3, range(200, 210), 1000, lambda t: t % 4)
        for p in d["profiles"]:
            p["offload"], p["consolidate"] = offload, consolidate
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
        _, end, ut = oracle.simulate(d["arrival_us"], d["true_len"], u, k, D, d["trace_off"], d["profiles"],
                                     d["trace_prof"], want_end=True, want_util=True)
        got = ctx.trace_utilization(torch.from_numpy(d["true_len"].view(np.int16)).to(DEV),
                                    torch.from_numpy(k.view(np.int64)).to(DEV), torch.from_numpy(end).to(DEV),
                                    d["trace_off"], d["profiles"],
                                    torch.from_numpy(d["trace_prof"].astype(np.uint16).view(np.int16)).to(DEV))
        got = got.cpu().numpy()
        assert (got[:, 0] == ut["gpu_busy_us"]).all()
        assert (got[:, 1] == ut["cpu_busy_us"]).all()
        assert ((got[:, 2] & 0xFFFFFFFF) == ut["gpu_batches"]).all()
        assert ((got[:, 2] >> 32) == ut["cpu_tasks"]).all()
        if offload:
            assert (ut["cpu_tasks"] > 0).any()
    # an empty trace reports zeros; a null array is an error
    z = torch.zeros(1, dtype=torch.int64, device=DEV)
    out = ctx.trace_utilization(z.view(torch.int16)[:1], z, z, np.array([0, 0]), d["profiles"][0])
    assert (out.cpu().numpy() == 0).all()
    with pytest.raises(rt.RtlmError):
        ctx.trace_utilization(None, z, z, np.array([0, 1]), d["profiles"][0])


@pytest.mark.gpu
@pytest.mark.parametrize("offload", [1, 0])
def test_trace_report_and_utilization_long_traces(ctx, offload):
    """NEXT-4 on traces beyond the 1024-task short path: two full paper ramps
    (11 280 tasks) beside 1000-task traces; report and utilization
    exact against the oracle (sorted responses / the event loop's accumulators)."""
    from oracle.offline import trace_report
    lex = oracle.Lexicon(configs.read_lexicon())
    dl = configs.traces(3, range(700, 702), 11280, lambda t: t % 4)
    ds = configs.traces(3, range(710, 713), 1000, lambda t: (t + 2) % 4)
    for dd in (dl, ds):
        for p in dd["profiles"]:
            p["offload"] = offload
    cat = {kk: np.concatenate([dl[kk], ds[kk]]) for kk in ("arrival_us", "true_len", "trace_prof")}
    toff = np.concatenate([dl["trace_off"], dl["trace_off"][-1] + ds["trace_off"][1:]]).astype(np.uint32)
    profs = dl["profiles"]
    u, k, D = [], [], []
    for dd in (dl, ds):
        f = oracle.rule_gen(lex, dd["data"], dd["offsets"])
        for t in range(len(dd["trace_off"]) - 1):
            lo, hi = int(dd["trace_off"][t]), int(dd["trace_off"][t + 1])
            lm = int(dd["trace_prof"][t])
            ut = oracle.predict(f[lo:hi], dd["regressors"][lm])
            kt, Dt = oracle.key(ut, f[lo:hi], profs[lm], r_us=dd["arrival_us"][lo:hi])
            u.append(ut), k.append(kt), D.append(Dt)
    u, k, D = np.concatenate(u), np.concatenate(k), np.concatenate(D)
    _, end, ut = oracle.simulate(cat["arrival_us"], cat["true_len"], u, k, D, toff, profs, cat["trace_prof"],
                                 want_end=True, want_util=True)
    rep = ctx.trace_report(torch.from_numpy(cat["arrival_us"]).to(DEV), torch.from_numpy(end).to(DEV), toff)
    rep = rep.cpu().numpy()
    want = trace_report(cat["arrival_us"], end, toff)
    assert (rep[:, 0] == want["max_resp_us"]).all()
    assert (rep[:, 1] == want["p95_resp_us"]).all()
    assert (rep[:, 2] == want["makespan_us"]).all()
    assert ((rep[:, 3] & 0xFFFFFFFF) == want["n"]).all() and want["n"][0] == 11280
    got = ctx.trace_utilization(torch.from_numpy(cat["true_len"].view(np.int16)).to(DEV),
                                torch.from_numpy(k.view(np.int64)).to(DEV), torch.from_numpy(end).to(DEV),
                                toff, profs, torch.from_numpy(cat["trace_prof"].astype(np.uint16).view(np.int16)).to(DEV))
    got = got.cpu().numpy()
    assert (got[:, 0] == ut["gpu_busy_us"]).all()
    assert (got[:, 1] == ut["cpu_busy_us"]).all()
    assert ((got[:, 2] & 0xFFFFFFFF) == ut["gpu_batches"]).all()
    assert ((got[:, 2] >> 32) == ut["cpu_tasks"]).all()
