"""Pins of oracle steps O3 (regression), O4 (priority key), O5 (order),
O6 (one-pass consolidation) and O7 (replay).

Expectations come from: SPEC worked examples (golden/spec_examples.json),
the hand-derived W1 schedule (golden/w1.json), closed forms (Lindley
recurrence S:418, single-task and batch latency S:384-393), brute force over
subsets (consolidation maximality) and over all 8! orders (Smith's and
Jackson's rules), and invariants.
"""
import itertools
import math
import random
import struct

import numpy as np
import pytest

import oracle
import rtgen
from rtgen import configs

BASE = dict(eta_us=50000, mu_us=80000, base_us=100000, setup_us=50000, xi_us=2000000, **{"lambda": 1.5},
            alpha=1.0, tau=35.0, u_max=40.0, C=11, b10=18, tightness=1, gamma=5, cores=4, policy="UP",
            consolidate=1, offload=1, raw_numerator=0)


def prof(**kw):
    p = dict(BASE)
    p.update(kw)
    return p


def unord32(k):
    b = int(k) & 0xFFFFFFFF
    bits = (b & 0x7FFFFFFF) if (b & 0x80000000) else (~b & 0xFFFFFFFF)
    return struct.unpack("<f", struct.pack("<I", bits))[0]


def feat_with_ntok(ntok):
    f = np.zeros((len(ntok), 8), np.uint16)
    f[:, 6] = ntok
    return f


# ------------------------------------------------------------------ O3
def test_regression_closed_forms():
    rng = np.random.default_rng(1)
    f = rng.integers(0, 40, size=(1000, 8)).astype(np.uint16)
    assert (oracle.predict(f, np.zeros(8)) == 0).all()                      # S:196 zero model
    g = np.float32(2.75)
    u = oracle.predict(f, [0, 0, 0, 0, 0, g, 0, 0])                         # S:197 route feature 4
    assert (u == g * f[:, 4].astype(np.float32)).all()
    assert (oracle.predict(f, [-1000, 0, 0, 0, 0, 0, 0, 0]) == 0).all()     # clamp at 0
    # fp32 fma chain vs exact fp64 value: |err| <= 8 ulp-ish, far inside 1e-5 relative
    p = configs.paper_lms()[0]
    reg = configs.regressor(p)
    u = oracle.predict(f, reg).astype(np.float64)
    exact = reg[0].astype(np.float64) + f[:, :7].astype(np.float64) @ reg[1:].astype(np.float64)
    assert np.all(np.abs(u - exact) <= 1e-6 * np.abs(exact))


def test_w1_regression(golden):
    w1 = golden("w1.json")
    f = np.zeros((8, 8), np.uint16)
    f[:, :7] = np.asarray(w1["feat_SYMVOP_ntok"])
    assert oracle.predict(f, configs.W1_REGRESSOR).tolist() == w1["u"]


# ------------------------------------------------------------------ O4
def test_priority_spec_examples(golden):
    for ex in golden("spec_examples.json")["priority"]:
        D_us = int(ex["D_s"] * 1e6)
        eta_us = int(round(ex["eta_s"] * 1e6))
        p = prof(policy=ex["policy"], eta_us=eta_us, alpha=ex.get("alpha", 1.0), u_max=ex.get("u_max", 40.0),
                 offload=0)
        k, D = oracle.key(np.float32([ex["u"]]), None, p, D_in=np.uint32([D_us]))
        assert (int(k[0]) >> 62) == 0
        v_per_us = unord32(k[0])
        assert math.isclose(v_per_us * 1e6, ex["p_per_s"], rel_tol=1e-6), ex["ref"]


def test_alpha_zero_equals_slack_order():
    """S:297 / S:336 / acceptance 11: alpha = 0 -> identical pop order."""
    rng = np.random.default_rng(2)
    for trial in range(100):
        n = int(rng.integers(2, 60))
        u = rng.uniform(1, 60, n).astype(np.float32)
        D = rng.integers(100000, 4000000, n).astype(np.uint32)
        k_up, _ = oracle.key(u, None, prof(policy="UP", alpha=0.0, offload=0), D_in=D)
        k_sl, _ = oracle.key(u, None, prof(policy="SLACK", offload=0), D_in=D)
        seg = np.uint32([0, n])
        assert (oracle.order(k_up, seg) == oracle.order(k_sl, seg)).all()


def test_numerator_monotonicity():
    """equal slack, normalized 0.2 vs 0.8 -> the 0.2 task strictly first (alpha = 1)."""
    # same eta*u requires same u; vary u_max instead? keep u equal and vary D to equalize slack:
    u = np.float32([8.0, 32.0])                         # un = 0.2, 0.8 with u_max = 40
    D = np.uint32([1000000 + 8 * 50000, 1000000 + 32 * 50000])  # both slack = 1 s
    k, _ = oracle.key(u, None, prof(offload=0), D_in=D)
    assert k[0] > k[1]


def test_offload_strictness():
    u = np.float32([35.0, np.nextafter(np.float32(35.0), np.float32(99)), 34.9, 35.001])
    k, _ = oracle.key(u, feat_with_ntok([10] * 4), prof())
    assert [int(x) >> 63 for x in k] == [0, 1, 0, 1]     # u = tau -> GPU
    k, _ = oracle.key(u, feat_with_ntok([10] * 4), prof(offload=0))
    assert all(int(x) >> 63 == 0 for x in k)


def test_baseline_orders():
    seg = np.uint32([0, 2])
    r = np.int64([1000000, 2000000])
    k, _ = oracle.key(np.float32([5, 9]), feat_with_ntok([3, 3]), prof(policy="FIFO", offload=0), r_us=r)
    assert oracle.order(k, seg).tolist() == [0, 1]
    k, _ = oracle.key(np.float32([5, 9]), None, prof(policy="LUF", offload=0), D_in=np.uint32([1, 1]))
    assert oracle.order(k, seg).tolist() == [0, 1]        # S:305 LUF: 5 first
    k, _ = oracle.key(np.float32([5, 9]), None, prof(policy="MUF", offload=0), D_in=np.uint32([1, 1]))
    assert oracle.order(k, seg).tolist() == [1, 0]        # MUF: 9 first
    k, _ = oracle.key(np.float32([5, 5]), None, prof(policy="EDF", offload=0), r_us=np.int64([0, 0]),
                      D_in=np.uint32([900, 500]))
    assert oracle.order(k, seg).tolist() == [1, 0]        # EDF: earlier deadline first
    k, _ = oracle.key(np.float32([5, 5]), None, prof(policy="LUF", offload=0), D_in=np.uint32([1, 1]))
    assert oracle.order(k, seg).tolist() == [0, 1]        # S:306 ties by lower id


def test_overdue_tier_and_deadline():
    # D = tightness * mu * ntok (mu 0.08, |J| = 10 -> 0.8 s; loose = 2x)
    u = np.float32([10, 30, 40, 2])
    f = feat_with_ntok([10, 10, 10, 10])
    k, D = oracle.key(u, f, prof(offload=0))
    assert D.tolist() == [800000] * 4
    k2, D2 = oracle.key(u, f, prof(offload=0, tightness=2))
    assert D2.tolist() == [1600000] * 4
    tiers = [(int(x) >> 62) & 1 for x in k]
    assert tiers == [0, 1, 1, 0]                           # slack = D - eta*u <= 1 µs -> overdue
    order = oracle.order(k, np.uint32([0, 4])).tolist()
    assert order == [2, 1, 0, 3]     # most negative slack first; then (1-u/40)/slk: 0.75/3e5 > 0.95/7e5


def test_w1_keys_and_one_pass_schedule(golden):
    w1 = golden("w1.json")
    c1 = configs.config1()
    lex = oracle.Lexicon(c1["lexicon"])
    f = oracle.rule_gen(lex, c1["data"], c1["offsets"])
    u = oracle.predict(f, c1["regressor"])
    k, D = oracle.key(u, f, c1["profile"])
    assert D.tolist() == w1["D_us"]
    assert [(int(x) >> 62) & 1 for x in k] == w1["overdue"]
    assert [int(x) >> 63 for x in k] == w1["cpu_class"]
    for i in range(8):
        slk = w1["slack_us"][i]
        if not w1["overdue"][i]:
            assert math.isclose(unord32(k[i]), (1 - w1["u"][i] / 40) / slk, rel_tol=1e-6)
        else:
            assert unord32(k[i]) == -slk
    s = oracle.schedule(k, u, np.uint32([0, 8]), c1["profile"])
    assert (s["perm"] + 1).tolist() == w1["key_order_1based"]
    assert s["nbatches"] == 1
    batch = sorted(range(8), key=lambda i: (s["batch_of"][i], s["slot_of"][i]))
    gpu = [i + 1 for i in batch if s["batch_of"][i] != 0xFFFFFFFF]
    assert [gpu] == w1["gpu_batches_1based"]
    assert s["core_of"][5] == 0 and s["batch_of"][5] == 0xFFFFFFFF


# ------------------------------------------------------------------ O6
def _single_queue_schedule(u, lam, C, b10, keys=None):
    n = len(u)
    if keys is None:  # priority order = input order (strictly decreasing keys)
        keys = np.arange(n, 0, -1).astype(np.uint64)
    return oracle.schedule(np.asarray(keys, np.uint64), np.float32(u), np.uint32([0, n]),
                           prof(**{"lambda": lam}, C=C, b10=b10, offload=0), cores=1)


def _batches(s, n):
    out = {}
    for i in range(n):
        if s["batch_of"][i] != 0xFFFFFFFF:
            out.setdefault(int(s["batch_of"][i]), []).append((int(s["slot_of"][i]), i))
    return [[i for _, i in sorted(v)] for _, v in sorted(out.items())]


def test_consolidate_spec_examples(golden):
    for ex in golden("spec_examples.json")["consolidate"]:
        s = _single_queue_schedule(ex["u"], ex["lambda"], ex["C"], ex["b10"])
        b = _batches(s, len(ex["u"]))
        if "first_batch_u" in ex:
            assert [ex["u"][i] for i in b[0]] == pytest.approx(ex["first_batch_u"]), ex["ref"]
        else:
            assert len(b[0]) == ex["first_batch_size"] and len(b[1]) == len(ex["u"]) - 4, ex["ref"]


def test_consolidation_bruteforce_maximal():
    """S:323 / acceptance 6: for random windows of size <= 12 the first
    batch is, among ALL subsets, the largest one that is a prefix of the
    ascending-u order, has every adjacent ratio <= lambda, and size <= C."""
    rng = random.Random(7)
    for trial in range(1000):
        n = rng.randint(1, 12)
        C = rng.randint(1, n)
        lam = rng.choice([1.0, 1.1, 1.5, 2.0])
        u = [float(np.float32(rng.choice([rng.uniform(1, 20), rng.randint(1, 6)]))) for _ in range(n)]
        s = _single_queue_schedule(u, lam, C, b10=int(math.ceil(10 * n / C)))  # one window holds all
        first = _batches(s, n)[0]
        order = sorted(range(n), key=lambda i: (u[i], i))
        best = None
        for mask in range(1, 1 << n):
            sub = [i for i in order if mask >> i & 1]
            if len(sub) > C or sub != order[:len(sub)]:
                continue
            if any(not (np.float32(u[sub[j]]) <= np.float32(lam) * np.float32(u[sub[j - 1]]))
                   for j in range(1, len(sub))):
                continue
            if best is None or len(sub) > len(best):
                best = sub
        assert first == best, (u, lam, C)


def test_one_pass_invariants():
    """batch sizes in [1, C], adjacent ratios <= lambda, every GPU task in
    exactly one batch, CPU routing strictly by tau, cores in range."""
    c2 = configs.config2(n=6000, gid0=123)
    lex = oracle.Lexicon(c2["lexicon"])
    f = oracle.rule_gen(lex, c2["data"], c2["offsets"])
    u = oracle.predict(f, c2["regressor"])
    for C, b10, lam in [(11, 18, 1.5), (33, 18, 1.5), (4, 10, 1.0), (7, 30, 3.0)]:
        p = dict(c2["profile"], C=C, b10=b10, **{"lambda": lam})
        k, D = oracle.key(u, f, p)
        s = oracle.schedule(k, u, np.uint32([0, 6000]), p)
        cpu = (k >> np.uint64(63)).astype(bool)
        assert ((u > np.float32(p["tau"])) == cpu).all()
        assert (s["batch_of"][cpu] == 0xFFFFFFFF).all() and (s["core_of"][cpu] < p["cores"]).all()
        b = _batches(s, 6000)
        assert sum(len(x) for x in b) == int((~cpu).sum())
        for x in b:
            assert 1 <= len(x) <= C
            us = u[x]
            assert (np.diff(us) >= 0).all()
            assert (us[1:] <= np.float32(lam) * us[:-1]).all()
        assert sorted(s["perm"].tolist()) == list(range(6000))
        assert (np.diff(k[s["perm"]].astype(np.float64)) <= 0).all()


# ------------------------------------------------------------------ O7
def _sim(r, ln, u, k, D, p, want_end=True):
    st, end = oracle.simulate(np.int64(r), np.uint16(ln), np.float32(u), np.uint64(k), np.uint32(D),
                              np.uint32([0, len(r)]), p, want_end=want_end)
    return st[0], end


def test_latency_closed_forms(golden):
    for ex in golden("spec_examples.json")["latency"]:
        n = len(ex["len"])
        if "CPU" in ex["what"]:
            p = prof(policy="FIFO", offload=1, tau=0.0)
            u = [1.0] * n
        else:
            p = prof(policy="FIFO", offload=0, consolidate=0, C=n)
            u = [1.0] * n
        k, D = oracle.key(np.float32(u), feat_with_ntok([1] * n), p, r_us=np.zeros(n, np.int64))
        st, end = _sim([0] * n, ex["len"], u, k, D, p)
        assert (end == int(round(ex["expect_s"] * 1e6))).all(), ex["ref"]


def test_lindley_recurrence():
    """FIFO, batch size 1, one executor -> start_i = max(r_i, end_{i-1})."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        n = 300
        r = np.cumsum(rng.integers(0, 3000000, n)).astype(np.int64)
        ln = rng.integers(1, 80, n).astype(np.uint16)
        p = prof(policy="FIFO", C=1, consolidate=0, offload=0)
        k, D = oracle.key(np.ones(n, np.float32), feat_with_ntok([5] * n), p, r_us=r)
        st, end = _sim(r, ln, np.ones(n), k, D, p)
        prev = 0
        for i in range(n):
            start = max(int(r[i]), prev)
            prev = start + p["setup_us"] + p["base_us"] + p["eta_us"] * int(ln[i])
            assert end[i] == prev
        assert st["sum_resp_us"] == int((end - r).sum())
        assert st["misses"] == int((end > r + D.astype(np.int64)).sum())


def test_single_task_flush():
    """one task in an empty system: response = flush delay + service.
    With no future arrivals the flush is immediate (DESIGN R-XI)."""
    p = prof(offload=0)
    k, D = oracle.key(np.float32([12.0]), feat_with_ntok([4]), p, r_us=np.int64([5000]))
    st, end = _sim([5000], [30], [12.0], k, D, p)
    assert end[0] - 5000 == p["setup_us"] + p["base_us"] + 30 * p["eta_us"]


def test_wait_interval_xi():
    """tasks arriving within xi are batched together; the oldest waits at most xi."""
    p = prof(policy="FIFO", offload=0, consolidate=0, C=4)
    r = [0, 1500000, 10_000_000]
    k, D = oracle.key(np.ones(3, np.float32), feat_with_ntok([5] * 3), p, r_us=np.int64(r))
    st, end = _sim(r, [10, 10, 10], [1, 1, 1], k, D, p)
    svc = p["setup_us"] + p["base_us"] + 10 * p["eta_us"]
    assert end[0] == end[1] == 2000000 + svc              # flushed together at 0 + xi
    assert end[2] == 10_000_000 + svc                     # last arrival: no future arrivals -> immediate


def test_replay_invariants_random():
    """Causality (response >= own service), conservation, determinism."""
    d = configs.traces(3, range(3), 400, lambda t: t % 4)
    lex = oracle.Lexicon(d["lexicon"])
    f = oracle.rule_gen(lex, d["data"], d["offsets"])
    for pol in ["FIFO", "EDF", "LUF", "MUF", "UP"]:
        for cons in (0, 1):
            for t in range(3):
                lo, hi = d["trace_off"][t], d["trace_off"][t + 1]
                p = dict(d["profiles"][d["trace_prof"][t]], policy=pol, consolidate=cons)
                u = oracle.predict(f[lo:hi], configs.regressor(p))
                k, D = oracle.key(u, f[lo:hi], p, r_us=d["arrival_us"][lo:hi])
                r, ln = d["arrival_us"][lo:hi], d["true_len"][lo:hi]
                st, end = _sim(r, ln, u, k, D, p)
                st2, end2 = _sim(r, ln, u, k, D, p)
                assert (end == end2).all() and st == st2
                cpu = (k >> np.uint64(63)).astype(bool)
                gsvc = p["setup_us"] + p["base_us"] + p["eta_us"] * ln.astype(np.int64)
                csvc = p["gamma"] * (p["base_us"] + p["eta_us"] * ln.astype(np.int64))
                assert (end - r >= np.where(cpu, csvc, gsvc)).all()
                assert st["n"] == hi - lo


def test_replay_equals_one_pass_when_all_arrive_at_zero():
    """DESIGN O7 invariant: with every arrival at 0, the replay's GPU batches equal O6's."""
    c2 = configs.config2(n=3000, gid0=9)
    lex = oracle.Lexicon(c2["lexicon"])
    f = oracle.rule_gen(lex, c2["data"], c2["offsets"])
    u = oracle.predict(f, c2["regressor"])
    for C, b10 in [(11, 18), (33, 16), (5, 10)]:
        p = dict(c2["profile"], C=C, b10=b10)
        k, D = oracle.key(u, f, p)
        s = oracle.schedule(k, u, np.uint32([0, 3000]), p)
        st, end = _sim(np.zeros(3000), c2["true_len"], u, k, D, p)
        gpu = s["batch_of"] != 0xFFFFFFFF
        # same partition of GPU tasks into batches, same batch order (end times increase per batch)
        b_end = {}
        for i in np.nonzero(gpu)[0]:
            b_end.setdefault(int(s["batch_of"][i]), set()).add(int(end[i]))
        assert all(len(v) == 1 for v in b_end.values())
        ends = [next(iter(b_end[b])) for b in sorted(b_end)]
        assert all(a < b for a, b in zip(ends, ends[1:]))


def test_bruteforce_config1_smith_jackson():
    """Config 1 brute force over all 8! orders (north_star): with exact predictions
    (u = true_len), C = 1, no offload, all r = 0:
      * LUF (= shortest processing time first) reaches the minimum mean response
        (Smith's rule) -- the paper's 'shorter execution times' intuition;
      * EDF reaches the minimum maximum lateness and zero misses whenever any
        order has zero misses (Jackson's rule) -- 'earlier deadlines'."""
    c1 = configs.config1()
    lex = oracle.Lexicon(c1["lexicon"])
    f = oracle.rule_gen(lex, c1["data"], c1["offsets"])
    ln = c1["true_len"].astype(np.int64)
    u = ln.astype(np.float32)
    for tight in (1, 2):
        p = dict(c1["profile"], C=1, consolidate=0, offload=0, tightness=tight)
        _, D = oracle.key(u, f, p)
        svc = p["setup_us"] + p["base_us"] + p["eta_us"] * ln
        best_sum, best_lmax, any_zero = None, None, False
        for perm in itertools.permutations(range(8)):
            t, s, lmax, miss = 0, 0, -10**18, 0
            for i in perm:
                t += int(svc[i])
                s += t
                lmax = max(lmax, t - int(D[i]))
                miss += t > int(D[i])
            best_sum = s if best_sum is None else min(best_sum, s)
            best_lmax = lmax if best_lmax is None else min(best_lmax, lmax)
            any_zero |= miss == 0
        for pol in ["LUF", "EDF", "UP"]:
            q = dict(p, policy=pol)
            k, _ = oracle.key(u, f, q, r_us=np.zeros(8, np.int64))
            st, end = _sim(np.zeros(8), ln, u, k, D, q)
            if pol == "LUF":
                assert st["sum_resp_us"] == best_sum
            if pol == "EDF":
                assert int((end - D.astype(np.int64)).max()) == best_lmax
                if any_zero:
                    assert st["misses"] == 0


@pytest.mark.parametrize("name", ["fig6.json", "fig7.json"])
def test_paper_toy_fixtures(golden, name):
    """Fig. 6 (EDF misses 2, LUF 3, EUDF 1) and Fig. 7 (P:269-285:
    oblivious batching misses 4, consolidation 2), instances found by
    scripts/find_fixtures.py and re-checked here through the oracle."""
    g = golden(name)
    n = len(g["len"])
    ln = np.asarray(g["len"], np.uint16)
    u = ln.astype(np.float32)
    D = (np.asarray(g["deadline_units"]) * g["unit_us"]).astype(np.uint32)
    for pname, want in g["misses"].items():
        p = g["profiles"][pname]
        k, _ = oracle.key(u, None, p, r_us=np.zeros(n, np.int64), D_in=D)
        st, _ = _sim(np.zeros(n), ln, u, k, D, p)
        assert st["misses"] == want, (name, pname)


def test_fixture_search_runs_fast():
    import subprocess, sys, time, tempfile, shutil, os
    t = time.time()
    # the search itself must finish well under 10 s
    out = subprocess.run([sys.executable, "-c", "import scripts.find_fixtures as f; import numpy as np; "
                          "p={k: dict(f.BASEP, policy=k) for k in ('EDF','LUF','UP')}; "
                          "print(f.search(5, {'EDF':2,'LUF':3,'UP':1}, p, np.random.default_rng(1)))"],
                         capture_output=True, text=True, cwd=os.path.dirname(os.path.dirname(__file__)))
    assert out.returncode == 0, out.stderr
    assert time.time() - t < 10


# ------------------------------------------------------------------ O6 CPU class (R-CORE)
def _cpu_fixture_inputs(fx):
    n = len(fx["perm"])
    key = np.zeros(n, np.uint64)
    u = np.zeros(n, np.float32)
    for j, i in enumerate(fx["perm"]):
        key[i] = (np.uint64(fx["cpu"][j]) << np.uint64(63)) | np.uint64(100 - j)
        u[i] = np.float32(fx["u"][j])
    p = prof(cores=fx["cores"], gamma=fx["gamma"], base_us=fx["base_us"], eta_us=fx["eta_us"], offload=1)
    return key, u, p


def _list_schedule_variant(fx, *, rnd="ceil", ties="low", base=True, fp64=False):
    """The hand table's rule and its plausible mis-readings (used only to show
    that the fixture tells them apart; the expected values are the table's)."""
    clocks = [0] * fx["cores"]
    out = []
    for j in range(len(fx["perm"])):
        if not fx["cpu"][j]:
            continue
        x = float(fx["eta_us"]) * float(np.float32(fx["u"][j])) if fp64 else \
            float(np.float32(fx["eta_us"]) * np.float32(fx["u"][j]))
        t = {"ceil": math.ceil(x), "trunc": int(x), "round": round(x)}[rnd]
        pred = fx["gamma"] * ((fx["base_us"] if base else 0) + t)
        lo = min(clocks)
        c = clocks.index(lo) if ties == "low" else len(clocks) - 1 - clocks[::-1].index(lo)
        clocks[c] += pred
        out.append(c)
    return out


def test_cpu_core_list_schedule_hand_tables(golden):
    """R-CORE pin: the oracle's core_of equals the hand-derived list schedules
    (tests/golden/cpu_cores.json) -- lowest-index ties, ceil of the single fp32
    product eta*u, base_us inside the latency, GPU-class tasks untouched."""
    for fx in golden("cpu_cores.json")["fixtures"]:
        key, u, p = _cpu_fixture_inputs(fx)
        n = len(u)
        s = oracle.schedule(key, u, np.uint32([0, n]), p)
        assert s["perm"].tolist() == fx["perm"], fx["name"]
        want = [st["core"] for st in fx["steps"]]
        got = [int(s["core_of"][fx["perm"][st["j"]]]) for st in fx["steps"]]
        assert got == want, fx["name"]
        for j, i in enumerate(fx["perm"]):
            if not fx["cpu"][j]:
                assert s["core_of"][i] == 0xFF and s["batch_of"][i] != 0xFFFFFFFF
            else:
                assert s["batch_of"][i] == 0xFFFFFFFF
        # the table's clocks are consistent with its own predicted latencies
        clocks = [0] * fx["cores"]
        for st in fx["steps"]:
            clocks[st["core"]] += st["pred"]
            assert clocks == st["clocks_after"], (fx["name"], st["j"])
    # each table separates the rule from its plausible mis-readings
    f3, f2 = golden("cpu_cores.json")["fixtures"]
    want3 = [st["core"] for st in f3["steps"]]
    want2 = [st["core"] for st in f2["steps"]]
    assert _list_schedule_variant(f3) == want3 and _list_schedule_variant(f2) == want2
    assert _list_schedule_variant(f3, ties="high") != want3
    assert _list_schedule_variant(f3, rnd="trunc") != want3
    assert _list_schedule_variant(f3, rnd="round") != want3
    assert _list_schedule_variant(f3, base=False) != want3
    assert _list_schedule_variant(f2, fp64=True) != want2


def test_cpu_core_choice_is_greedy_minimum():
    """R-CORE checker on large random queues: replay the oracle's core_of in key
    order, rebuilding each core's predicted clock from the definition
    gamma*(base + ceil(fp32(eta*u))); every choice must be a core of minimal
    clock, the lowest-index one among ties.  Includes crafted ties (equal u)."""
    rng = np.random.default_rng(11)
    for trial in range(6):
        n = int(rng.integers(50, 3000))
        cores = int(rng.integers(1, 9))
        u = np.where(rng.random(n) < 0.3, np.float32(rng.integers(1, 4)), rng.uniform(0.1, 200, n)).astype(np.float32)
        cpu = rng.random(n) < 0.7
        key = (cpu.astype(np.uint64) << np.uint64(63)) | rng.permutation(n).astype(np.uint64)
        p = prof(cores=cores, gamma=int(rng.integers(1, 6)), base_us=int(rng.integers(0, 200000)),
                 eta_us=int(rng.integers(1, 120000)), offload=1)
        s = oracle.schedule(key, u, np.uint32([0, n]), p)
        clocks = [0] * cores
        seen = 0
        for i in s["perm"]:
            if not cpu[i]:
                assert s["core_of"][i] == 0xFF
                continue
            c = int(s["core_of"][i])
            lo = min(clocks)
            assert clocks[c] == lo and clocks.index(lo) == c, (trial, seen)
            eu = np.float32(p["eta_us"]) * np.float32(u[i])
            clocks[c] += p["gamma"] * (p["base_us"] + math.ceil(float(eu)))
            seen += 1
        assert seen == int(cpu.sum())


def test_cpu_core_choice_invariant_under_gamma():
    """gamma scales every predicted latency by the same factor, so the argmin
    choices (ties included) cannot change with gamma."""
    c2 = configs.config2(n=4000, gid0=77)
    lex = oracle.Lexicon(c2["lexicon"])
    f = oracle.rule_gen(lex, c2["data"], c2["offsets"])
    u = oracle.predict(f, c2["regressor"])
    p = dict(c2["profile"], tau=float(np.quantile(u, 0.5)))
    k, _ = oracle.key(u, f, p)
    ref = oracle.schedule(k, u, np.uint32([0, 4000]), dict(p, gamma=1))["core_of"]
    for g in (2, 5, 7):
        assert (oracle.schedule(k, u, np.uint32([0, 4000]), dict(p, gamma=g))["core_of"] == ref).all()


def _moore_hodgson(p_us, d_us):
    """Minimum number of late jobs on one machine, all released at 0
    (Moore-Hodgson): EDF order; whenever the running completion exceeds the
    current job's due date, drop the longest job scheduled so far."""
    import heapq
    t, heap, late = 0, [], 0
    for i in sorted(range(len(p_us)), key=lambda i: d_us[i]):
        t += p_us[i]
        heapq.heappush(heap, -p_us[i])
        if t > d_us[i]:
            t += heapq.heappop(heap)
            late += 1
    return late


def test_bruteforce_misses_up_vs_moore_hodgson(golden):
    """Config 1 (C = 1, no offload, exact predictions, all r = 0) and the Fig. 6
    instance: the minimum number of misses over ALL orders (brute force) equals
    Moore-Hodgson's optimum; the replay's miss count for the UP order equals the
    brute-force evaluator's count for that same order; UP never beats the
    optimum.  Paper intuition (Fig. 6): on the Fig. 6 instance EUDF
    (= UP) misses one deadline, and that is the optimum.  On config 1 the
    paper's deadlines d = mu*|J| are shorter than almost every service time, so
    UP's count is reported next to the optimum (not gated beyond >= optimum)."""
    c1 = configs.config1()
    lex = oracle.Lexicon(c1["lexicon"])
    f = oracle.rule_gen(lex, c1["data"], c1["offsets"])
    ln = c1["true_len"].astype(np.int64)
    u = ln.astype(np.float32)
    report = {}
    for tight in (1, 2, 4, 8):
        p = dict(c1["profile"], C=1, consolidate=0, offload=0, tightness=tight)
        _, D = oracle.key(u, f, p)
        svc = [int(x) for x in p["setup_us"] + p["base_us"] + p["eta_us"] * ln]
        Dl = [int(x) for x in D]

        def misses(order):
            t, m = 0, 0
            for i in order:
                t += svc[i]
                m += t > Dl[i]
            return m
        best = min(misses(o) for o in itertools.permutations(range(8)))
        assert _moore_hodgson(svc, Dl) == best
        q = dict(p, policy="UP")
        k, _ = oracle.key(u, f, q, r_us=np.zeros(8, np.int64))
        st, end = _sim(np.zeros(8), ln, u, k, D, q)
        order = sorted(range(8), key=lambda i: end[i])
        assert int(st["misses"]) == misses(order)
        assert int(st["misses"]) >= best
        report[tight] = (int(st["misses"]), best)
    print("config-1 UP misses vs optimum by tightness:", report)
    g = golden("fig6.json")
    ln6 = [int(x) * g["unit_us"] for x in g["len"]]
    d6 = [int(x) * g["unit_us"] for x in g["deadline_units"]]
    best6 = min(sum(t > d6[i] for t, i in zip(itertools.accumulate(ln6[j] for j in o), o))
                for o in itertools.permutations(range(5)))
    assert best6 == _moore_hodgson(ln6, d6) == g["misses"]["UP"] == 1
