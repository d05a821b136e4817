"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bar (north_star): features, keys, orders, batch/core
assignments, end times and miss counts bit-exact; u bit-exact too (same fp32
operation sequence; the 1e-5 relative tolerance of north_star is asserted as
the outer bound).
"""
import numpy as np
import pytest

import oracle
import rtgen
from rtgen import configs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2309_06619_b200 as rt  # noqa: E402

DEV = torch.device("cuda", 0)
U32 = np.uint32


def dev(a):
    a = np.ascontiguousarray(a)
    view = {np.dtype(np.uint32): np.int32, np.dtype(np.uint16): np.int16, np.dtype(np.uint64): np.int64}
    if a.dtype in view:
        a = a.view(view[a.dtype])
    return torch.from_numpy(a).to(DEV)


def host(t, dtype):
    return t.cpu().numpy().view(dtype)


@pytest.fixture(scope="module")
def ctx_v1():
    return rt.Context(configs.read_lexicon(), 0)


@pytest.fixture(scope="module")
def ctx_min():
    return rt.Context(configs.read_lexicon(configs.LEX_MIN), 0)


@pytest.fixture(scope="module")
def lex_v1():
    return oracle.Lexicon(configs.read_lexicon())


def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


def edge_texts():
    rng = np.random.default_rng(11)
    t = ["", " ", "?", "a", "n't", "don't", "DON'T STOP!!", "What's", "x" * 40, "stuffing" * 3, "'s's's",
         "Why art? How art? Tell art?", "a, b, c, d", "a,, b", "cats, and dogs", "bats's", "flies'",
         "\t\n\x0b\x0c\r", "caf\xe9 na\xefve", "abcdefghijklmnopqrsing", "abcdefghijklmnopqing", "abcdefghijklmnoping",
         "abcdefghijklmnopqrs's", "history" * 3 + "'s", "John saw a boy in the park with a telescope.",
         "What are the causes and consequences of poverty in developing countries?"]
    for _ in range(300):  # random bytes over the whole 0..255 range
        t.append(bytes(rng.integers(0, 256, size=int(rng.integers(0, 60)), dtype=np.uint8)))
    for _ in range(300):  # random printable soup with apostrophes and punctuation
        alphabet = np.frombuffer(b"abcdeSTUVW'0123 ,.?!;-\t", dtype=np.uint8)
        t.append(bytes(rng.choice(alphabet, size=int(rng.integers(0, 80)))))
    t.append("stuff " * 9000)            # > 32 KB staging tile: slow path
    t.append("and " * 70000)             # u16 saturation of ntok
    return t


@pytest.mark.parametrize("lexname", ["v1", "min"])
def test_score_edge_cases(lexname, ctx_v1, ctx_min):
    ctx = ctx_v1 if lexname == "v1" else ctx_min
    lex = oracle.Lexicon(configs.read_lexicon() if lexname == "v1" else configs.read_lexicon(configs.LEX_MIN))
    data, off = rtgen.pack_texts(edge_texts())
    feat = ctx.score(dev(data), dev(off))
    torch.cuda.synchronize()
    got = host(feat, np.uint16)
    want = oracle.rule_gen(lex, data, off)
    bad = np.nonzero((got != want).any(1))[0]
    assert len(bad) == 0, [(int(i), bytes(data[off[i]:off[i + 1]])[:60], got[i].tolist(), want[i].tolist())
                           for i in bad[:5]]
    assert ctx.flags() & 1  # saturation was flagged


def _score_all(ctx, lex, d, prof, reg, arrival=None):
    out = ctx.score_key(dev(d["data"]), dev(d["offsets"]), reg, prof,
                        arrival=None if arrival is None else dev(arrival), want_feat=True)
    torch.cuda.synchronize()
    f = oracle.rule_gen(lex, d["data"], d["offsets"])
    u = oracle.predict(f, reg)
    k, D = oracle.key(u, f, prof, r_us=arrival)
    return out, f, u, k, D


def test_score_key_parity_ragged(ctx_v1, lex_v1):
    """50 001 requests: many tiles plus a ragged tail."""
    d = configs.config2(n=50001, gid0=777)
    out, f, u, k, D = _score_all(ctx_v1, lex_v1, d, d["profile"], d["regressor"])
    assert (host(out["feat"], np.uint16) == f).all()
    gu = out["u"].cpu().numpy()
    assert np.all(np.abs(gu - u) <= 1e-5 * np.abs(u))
    assert (gu.view(U32) == u.view(U32)).all()
    assert (host(out["key"], np.uint64) == k).all()
    assert (host(out["D"], U32) == D).all()
    # unfused calls agree with the fused one
    feat = ctx_v1.score(dev(d["data"]), dev(d["offsets"]))
    u2 = ctx_v1.predict(feat, d["regressor"])
    k2, D2 = ctx_v1.key(u2, d["profile"], feat=feat)
    torch.cuda.synchronize()
    assert (host(feat, np.uint16) == f).all()
    assert (u2.cpu().numpy().view(U32) == u.view(U32)).all()
    assert (host(k2, np.uint64) == k).all() and (host(D2, U32) == D).all()


@pytest.mark.parametrize("policy", ["FIFO", "EDF", "LUF", "MUF", "SLACK", "UP"])
@pytest.mark.parametrize("variant", ["plain", "loose_raw_nooffload"])
def test_key_policies(ctx_v1, lex_v1, policy, variant):
    d = configs.traces(3, range(2), 1000, lambda t: t % 4)
    prof = dict(d["profiles"][0], policy=policy)
    if variant != "plain":
        prof.update(tightness=2, raw_numerator=1, offload=0, alpha=0.3)
    out, f, u, k, D = _score_all(ctx_v1, lex_v1, d, prof, d["regressors"][0], arrival=d["arrival_us"])
    assert (host(out["key"], np.uint64) == k).all()
    assert (host(out["D"], U32) == D).all()


def _check_schedule(g, s, nseg):
    assert (host(g["perm"], U32) == s["perm"]).all(), "perm"
    assert (host(g["batch_of"], U32) == s["batch_of"]).all(), "batch_of"
    assert (g["slot_of"].cpu().numpy() == s["slot_of"]).all(), "slot_of"
    assert (g["core_of"].cpu().numpy() == s["core_of"]).all(), "core_of"
    assert (host(g["seg_batch_off"], U32) == s["seg_batch_off"]).all(), "seg_batch_off"


@pytest.mark.parametrize("C,b10,lam,cores", [(11, 18, 1.5, 4), (33, 18, 1.5, 4), (4, 10, 1.0, 1), (24, 30, 2.0, 32),
                                             (1, 10, 1.5, 7)])
def test_schedule_many_small_queues(ctx_v1, lex_v1, C, b10, lam, cores):
    rng = np.random.default_rng(C * 100 + b10)
    sizes = [0, 1, 2, 2048, 37] + [int(x) for x in rng.integers(0, 700, 60)]
    seg = np.concatenate([[0], np.cumsum(sizes)]).astype(U32)
    d = configs.config2(n=int(seg[-1]), gid0=5000 + C)
    prof = dict(d["profile"], C=C, b10=b10, **{"lambda": lam}, cores=cores)
    out, f, u, k, D = _score_all(ctx_v1, lex_v1, d, prof, d["regressor"])
    g = ctx_v1.schedule(out["key"], out["u"], seg, prof)
    torch.cuda.synchronize()
    s = oracle.schedule(k, u, seg, prof)
    _check_schedule(g, s, len(sizes))


@pytest.mark.parametrize("n", [2049, 30000])
def test_schedule_big_queue(ctx_v1, lex_v1, n):
    d = configs.config2(n=n, gid0=90000)
    for pol in ["UP", "FIFO"]:
        prof = dict(d["profile"], policy=pol)
        out, f, u, k, D = _score_all(ctx_v1, lex_v1, d, prof, d["regressor"], arrival=np.zeros(n, np.int64))
        seg = np.asarray([0, n], U32)
        g = ctx_v1.schedule(out["key"], out["u"], seg, prof)
        torch.cuda.synchronize()
        s = oracle.schedule(k, u, seg, prof)
        _check_schedule(g, s, 1)


@pytest.mark.parametrize("C,b10,lam,cores", [(11, 18, 1.5, 4), (33, 18, 1.5, 4), (11, 10, 1.5, 4), (33, 30, 1.5, 2),
                                             (5, 20, 1.0, 1), (24, 13, 3.0, 8), (1, 10, 1.5, 4), (11, 18, 1.05, 32)])
def test_schedule_big_queue_params(ctx_v1, lex_v1, C, b10, lam, cores):
    """The parallel consolidation path (queues > 2048) against O6 for window
    shapes K = m - C from 0 to 66 and lambda from 1.0 (cuts everywhere) to 3.0."""
    n = 20011
    d = configs.config2(n=n, gid0=424242 + C)
    prof = dict(d["profile"], C=C, b10=b10, **{"lambda": lam}, cores=cores)
    out, f, u, k, D = _score_all(ctx_v1, lex_v1, d, prof, d["regressor"])
    seg = np.asarray([0, n], U32)
    g = ctx_v1.schedule(out["key"], out["u"], seg, prof)
    torch.cuda.synchronize()
    _check_schedule(g, oracle.schedule(k, u, seg, prof), 1)


def test_schedule_big_queue_no_offload_and_tiny_gpu_class(ctx_v1, lex_v1):
    """All-GPU queue, and a queue whose GPU class is smaller than the carry K."""
    n = 5000
    d = configs.config2(n=n, gid0=777777)
    for prof in [dict(d["profile"], offload=0), dict(d["profile"], tau=6.0, C=33, b10=30)]:
        out, f, u, k, D = _score_all(ctx_v1, lex_v1, d, prof, d["regressor"])
        seg = np.asarray([0, n], U32)
        g = ctx_v1.schedule(out["key"], out["u"], seg, prof)
        torch.cuda.synchronize()
        _check_schedule(g, oracle.schedule(k, u, seg, prof), 1)


def test_schedule_mixed_big_and_small(ctx_v1, lex_v1):
    sizes = [100, 5000, 0, 3000, 7]
    seg = np.concatenate([[0], np.cumsum(sizes)]).astype(U32)
    d = configs.config2(n=int(seg[-1]), gid0=123456)
    out, f, u, k, D = _score_all(ctx_v1, lex_v1, d, d["profile"], d["regressor"])
    g = ctx_v1.schedule(out["key"], out["u"], seg, d["profile"])
    torch.cuda.synchronize()
    _check_schedule(g, oracle.schedule(k, u, seg, d["profile"]), len(sizes))


def _replay_case(ctx, lex, d, overrides, want_end=True):
    nt = len(d["trace_off"]) - 1
    profs = [dict(p, **overrides) for p in d["profiles"]]
    u = np.zeros(len(d["arrival_us"]), np.float32)
    k = np.zeros(len(u), np.uint64)
    D = np.zeros(len(u), U32)
    f = oracle.rule_gen(lex, d["data"], d["offsets"])
    gpu_u, gpu_k, gpu_D = [], [], []
    for t in range(nt):
        lo, hi = int(d["trace_off"][t]), int(d["trace_off"][t + 1])
        p = profs[int(d["trace_prof"][t])]
        reg = d["regressors"][int(d["trace_prof"][t])]
        u[lo:hi] = oracle.predict(f[lo:hi], reg)
        k[lo:hi], D[lo:hi] = oracle.key(u[lo:hi], f[lo:hi], p, r_us=d["arrival_us"][lo:hi])
    st, end = oracle.simulate(d["arrival_us"], d["true_len"], u, k, D, d["trace_off"], profs, d["trace_prof"],
                              want_end=want_end)
    gs, gend = ctx.simulate(dev(d["arrival_us"]), dev(d["true_len"]), dev(u), dev(k), dev(D), d["trace_off"], profs,
                            dev(d["trace_prof"]), want_end=want_end)
    torch.cuda.synchronize()
    g = rt.decode_stats(gs)
    assert (g == st).all(), [(i, g[i], st[i]) for i in np.nonzero(g != st)[0][:3]]
    if want_end:
        assert (gend.cpu().numpy() == end).all()
    return st


@pytest.mark.parametrize("ov", [{}, {"consolidate": 0}, {"offload": 0}, {"policy": "FIFO", "consolidate": 0,
                                                                          "offload": 0},
                                {"policy": "LUF"}, {"policy": "MUF"}, {"policy": "EDF"}, {"tightness": 2},
                                {"b10": 30, "lambda": 1.1}, {"cores": 1}, {"xi_us": 0}])
def test_replay_parity(ctx_v1, lex_v1, ov):
    d = configs.traces(3, range(40, 56), 1000, lambda t: t % 4)
    _replay_case(ctx_v1, lex_v1, d, ov)


def test_replay_sizes_and_heavy_load(ctx_v1, lex_v1):
    # trace sizes 1 and 1024 and a 16x arrival-rate overload
    d = configs.traces(5, range(8), 1024, lambda t: t % 4, beta0=160, step=16, beta_max=2400)
    _replay_case(ctx_v1, lex_v1, d, {})
    d1 = configs.traces(5, range(3), 1, lambda t: t % 4)
    _replay_case(ctx_v1, lex_v1, d1, {})


def test_reduce_stats(ctx_v1):
    rng = np.random.default_rng(3)
    nt = 5000
    raw = np.zeros((nt, 2), np.int64)
    raw[:, 0] = rng.integers(0, 2**40, nt)
    n = rng.integers(0, 1025, nt).astype(np.uint64)
    m = rng.integers(0, 1025, nt).astype(np.uint64)
    raw[:, 1] = (n | (m << np.uint64(32))).view(np.int64)
    grp = rng.integers(0, 7, nt).astype(np.uint16)
    sums = ctx_v1.reduce_stats(dev(raw), dev(grp), 7)
    torch.cuda.synchronize()
    for gi in range(7):
        sel = grp == gi
        assert sums[gi, 0].item() == int(raw[sel, 0].sum())
        assert sums[gi, 1].item() == int(n[sel].sum()) and sums[gi, 2].item() == int(m[sel].sum())


def test_errors(ctx_v1):
    with pytest.raises(rt.RtlmError, match="RT_ELEXICON"):
        rt.Context("bogus:\nx\n", 0)
    p = dict(configs.paper_lms()[0], **{"lambda": 0.5})
    u = torch.zeros(4, device=DEV)
    with pytest.raises(rt.RtlmError, match="lambda"):
        ctx_v1.key(u, p, D_in=torch.zeros(4, dtype=torch.int32, device=DEV))
    p = dict(configs.paper_lms()[0], C=200)
    with pytest.raises(rt.RtlmError, match="RT_EINVAL"):
        ctx_v1.key(u, p, D_in=torch.zeros(4, dtype=torch.int32, device=DEV))


@pytest.mark.slow
def test_config2_full_size(ctx_v1, lex_v1):
    """BASELINE configs[1] at full size (2^20 requests, one queue), in the bench's
    launch configuration: score_key + schedule, everything compared with the oracle."""
    d = configs.config2()
    out, f, u, k, D = _score_all(ctx_v1, lex_v1, d, d["profile"], d["regressor"])
    assert (host(out["feat"], np.uint16) == f).all()
    assert (out["u"].cpu().numpy().view(U32) == u.view(U32)).all()
    assert (host(out["key"], np.uint64) == k).all()
    seg = np.asarray([0, len(u)], U32)
    g = ctx_v1.schedule(out["key"], out["u"], seg, d["profile"])
    torch.cuda.synchronize()
    _check_schedule(g, oracle.schedule(k, u, seg, d["profile"]), 1)


def test_config4_shape_parity(ctx_v1, lex_v1):
    """BASELINE configs[3] shape: traces of 1024 requests (65 536 per job, 8 192
    per rank); a sample of one rank's shard replayed against the oracle."""
    d = configs.config4_shard(rank=3, world=8, n_traces=65536, per_trace=1024)
    sub = {k: d[k] for k in ("profiles", "regressors", "lexicon")}
    # take the first 24 traces of the shard (bytes/offsets sliced consistently)
    nt = 24
    lo_req, hi_req = 0, int(d["trace_off"][nt])
    b0, b1 = int(d["offsets"][lo_req]), int(d["offsets"][hi_req])
    sub.update(data=d["data"][b0:b1], offsets=(d["offsets"][:hi_req + 1] - b0).astype(np.uint32),
               arrival_us=d["arrival_us"][:hi_req], true_len=d["true_len"][:hi_req],
               trace_off=d["trace_off"][:nt + 1], trace_prof=d["trace_prof"][:nt])
    _replay_case(ctx_v1, lex_v1, sub, {})


@pytest.mark.parametrize("point", [
    {"policy": "FIFO", "consolidate": 0, "offload": 0}, {"policy": "EDF", "consolidate": 0, "offload": 0},
    {"policy": "LUF", "consolidate": 0, "offload": 0}, {"policy": "MUF", "consolidate": 0, "offload": 0},
    {"policy": "UP", "consolidate": 0, "offload": 0}, {"policy": "UP", "consolidate": 1, "offload": 0},
    {"policy": "UP", "alpha": 0.0}, {"policy": "UP", "alpha": 2.0}, {"policy": "UP", "b10": 10},
    {"policy": "UP", "b10": 30}, {"tightness": 2}])
@pytest.mark.parametrize("mult", [0.25, 4.0, 32.0])
def test_config5_sweep_points(ctx_v1, lex_v1, point, mult):
    """BASELINE configs[4]: arrival-rate multipliers x policy / consolidation /
    offload / alpha / b / tightness points."""
    d = configs.traces(5, range(int(mult * 100), int(mult * 100) + 8), 1000, lambda t: t % 4,
                       beta0=10 * mult, step=1 * mult, beta_max=150 * mult)
    _replay_case(ctx_v1, lex_v1, d, point)


def test_config5_grid_as_one_replay(ctx_v1, lex_v1):
    """bench.py's config-5 leg replays the whole sweep grid in ONE rt_simulate:
    the same traces repeated per point, with per-trace profile index point*4 + LM
    and the point's arrivals (rate multiplier).  Stats per (point, LM) through
    rt_reduce_stats; everything against the oracle, point by point."""
    base = configs.config5_base(900, per_lm=2)
    pts = [p for p in configs.config5_points() if p["name"] in ("FIFO/t1", "UP+C+O/t2", "alpha=0.5", "b=2.5")]
    pts = [dict(p, mult=m) for p, m in zip(pts, (0.25, 32.0, 8.0, 8.0))]
    npt, n, nt = len(pts), len(base["arrival_us"]), len(base["trace_off"]) - 1
    d = dict(base)
    d["data"] = np.concatenate([base["data"]] * npt)
    tot = int(base["offsets"][-1])
    d["offsets"] = np.concatenate([base["offsets"][:-1].astype(np.uint64) + i * tot for i in range(npt)]
                                  + [np.asarray([npt * tot], np.uint64)]).astype(np.uint32)
    d["arrival_us"] = np.concatenate([configs.config5_arrivals(base, p["mult"]) for p in pts])
    d["true_len"] = np.tile(base["true_len"], npt)
    d["trace_off"] = (np.arange(npt * nt + 1, dtype=np.uint64) * int(base["trace_off"][1])).astype(U32)
    d["trace_prof"] = np.concatenate([base["trace_prof"] + 4 * i for i in range(npt)]).astype(np.uint16)
    d["profiles"] = [dict(p, **pt["overrides"]) for pt in pts for p in base["profiles"]]
    d["regressors"] = [r for _ in pts for r in base["regressors"]]
    st = _replay_case(ctx_v1, lex_v1, d, {})
    gsums = ctx_v1.reduce_stats(dev(st.view(np.int64).reshape(-1, 2)), dev(d["trace_prof"]), npt * 4)
    torch.cuda.synchronize()
    for g in range(npt * 4):
        sel = d["trace_prof"] == g
        assert gsums[g, 0].item() == int(st["sum_resp_us"][sel].sum())
        assert gsums[g, 2].item() == int(st["misses"][sel].sum())


def test_score_stream_boundaries(ctx_v1, lex_v1):
    """K1 streams 512-byte chunks: words and clitics across chunk boundaries, runs
    longer than one and two chunks, requests splitting a word, and requests with
    thousands of tokens (many 32-token rule batches, carries across chunks)."""
    t = []
    for pad in list(range(500, 516)) + list(range(985, 1000)) + list(range(1012, 1030)):
        t.append("a" * pad + " don't stop.")  # a word (with clitic) straddling a chunk boundary
    t += ["x" * 600 + "n't", "y" * 1100 + "'s and stuff", "history" * 100, "Why" + "z" * 530 + "?",
          "q" * 511 + " " + "r" * 513 + "'ll"]
    t += ["ab", "cd", "n't", "s", "'s", "", "", "ing", "edges"]  # adjacent requests split words
    t += ["a, b, c. " * 700, "What causes art? " * 400, "John saw a boy in the park with a telescope. " * 150]
    rng = np.random.default_rng(5)
    words = ["the", "art", "of", "and", "stuff", "bats", "what", "why", "flies", "like", "sand", ",", ".", "?",
             "don't", "it's", "we've", "history", "\xe9"]
    for _ in range(200):
        t.append(" ".join(rng.choice(words, size=int(rng.integers(1, 400)))))
    data, off = rtgen.pack_texts(t)
    feat = ctx_v1.score(dev(data), dev(off))
    torch.cuda.synchronize()
    got, want = host(feat, np.uint16), oracle.rule_gen(lex_v1, data, off)
    bad = np.nonzero((got != want).any(1))[0]
    assert len(bad) == 0, [(int(i), got[i].tolist(), want[i].tolist()) for i in bad[:5]]


def test_score_pool_boundaries(ctx_v1, lex_v1):
    """K1 tokenizes whole warp tasks (32 requests) into a per-warp pool of up to
    16 tasks / 16384 tokens before the rule pass: tasks of 2-16 KB fill a pool
    after a few tasks (the next task waits for the following pool), tasks above
    16 KB take the per-lane byte path, and empty requests sit between, before
    and after requests with tokens (also at pool ends)."""
    d = configs.config2(n=6000, gid0=99)
    data, off = d["data"], d["offsets"]
    reqs = [bytes(data[off[i]:off[i + 1]]) for i in range(len(off) - 1)]
    rng = np.random.default_rng(17)
    t, k = [], 0
    while k < len(reqs) - 40:
        kind = rng.integers(0, 4)
        if kind == 0:  # a task of ~2-16 KB: 32 requests of 1-7 generator requests each
            for _ in range(32):
                m = int(rng.integers(1, 8))
                t.append(b" ".join(reqs[k:k + m]))
                k += m
        elif kind == 1:  # empty requests around short ones
            for _ in range(32):
                t.append(b"" if rng.random() < 0.5 else reqs[k])
                k += 1
        elif kind == 2:  # one task above 16 KB (byte path) or just below it
            big = int(rng.integers(14000, 19000))
            chunk = b" ".join(reqs[k:k + 260])[:big]
            k += 260
            t += [chunk[i * len(chunk) // 32:(i + 1) * len(chunk) // 32] for i in range(32)]
        else:
            t += reqs[k:k + 32]
            k += 32
    t += [b""] * 40
    data2, off2 = rtgen.pack_texts(t)
    feat = ctx_v1.score(dev(data2), dev(off2))
    torch.cuda.synchronize()
    got, want = host(feat, np.uint16), oracle.rule_gen(lex_v1, data2, off2)
    bad = np.nonzero((got != want).any(1))[0]
    assert len(bad) == 0, [(int(i), got[i].tolist(), want[i].tolist()) for i in bad[:5]]


def test_score_chunk_boundaries_random_runs(ctx_v1, lex_v1):
    """K1 stages 1 KB chunks after the previous chunk's last 32 bytes: runs of
    1-48 bytes (lexicon words with suffixes and clitics, upper case, digits)
    at every offset around the chunk boundaries, including runs that started
    more than 32 bytes before a chunk (carried as the 24-byte run ending where
    they end) and runs that end exactly at a chunk end."""
    rng = np.random.default_rng(23)
    stems = ["history", "stuff", "bank", "john", "what", "why", "and", "or", "flies", "like", "art", "poverty",
             "x" * 14, "y" * 16, "z" * 20, "abcdefghijklmnopqrstuvwxyzabcdefghij", "a"]
    tails = ["", "s", "es", "ed", "ing", "'s", "n't", "'ll", "'re", "'ve", "'m", "'d", "s's", "ing's"]
    t = []
    for _ in range(96 * 32):
        parts = []
        for _ in range(int(rng.integers(1, 40))):
            w = rng.choice(stems) + rng.choice(tails)
            if rng.random() < 0.1:
                w = w.upper()
            if rng.random() < 0.05:
                w = w * int(rng.integers(2, 5))  # long runs
            parts.append(w)
            parts.append(rng.choice([" ", "  ", ", ", ". ", "? ", "", "\t"]))
        t.append("".join(parts)[: int(rng.integers(0, 400))])
    data, off = rtgen.pack_texts(t)
    feat = ctx_v1.score(dev(data), dev(off))
    torch.cuda.synchronize()
    got, want = host(feat, np.uint16), oracle.rule_gen(lex_v1, data, off)
    bad = np.nonzero((got != want).any(1))[0]
    assert len(bad) == 0, [(int(i), bytes(data[off[i]:off[i + 1]])[:80], got[i].tolist(), want[i].tolist())
                           for i in bad[:5]]


def test_score_runs_longer_than_32_bytes(ctx_v1, lex_v1):
    """A run's length comes from a 32-bit window of the stop mask; runs of
    28-72 bytes (plain, with a suffix, with a clitic) at every byte alignment,
    so their ends fall in every bit of the following stop words."""
    t = []
    for L in range(28, 73):
        for pre in range(0, 33):
            for tail in ("", "ing", "'s", "n't"):
                t.append(" " * pre + "b" * L + tail + " and stuff.")
    data, off = rtgen.pack_texts(t)
    feat = ctx_v1.score(dev(data), dev(off))
    torch.cuda.synchronize()
    got, want = host(feat, np.uint16), oracle.rule_gen(lex_v1, data, off)
    bad = np.nonzero((got != want).any(1))[0]
    assert len(bad) == 0, [(int(i), bytes(data[off[i]:off[i + 1]])[:80], got[i].tolist(), want[i].tolist())
                           for i in bad[:5]]


@pytest.mark.parametrize("ctas", [1, 3])
def test_score_few_ctas_many_pools(lex_v1, ctas):
    """rt_set_sm_limit(1 / 3): 32 / 96 warps take all 1 563 tasks of a 50 001-request
    queue, so every warp fills dozens of 8-task pools in turn (the pool loop, the
    pending task carried into the next pool, the self-resetting work counter
    over repeated launches)."""
    ctx = rt.Context(configs.read_lexicon(), 0)
    ctx.set_sm_limit(ctas)
    d = configs.config2(n=50001, gid0=31337)
    want = oracle.rule_gen(lex_v1, d["data"], d["offsets"])
    for _ in range(2):
        feat = ctx.score(dev(d["data"]), dev(d["offsets"]))
        torch.cuda.synchronize()
        got = host(feat, np.uint16)
        assert (got == want).all()


def test_score_decreasing_offsets(ctx_v1, lex_v1):
    """Offsets that decrease: those requests score as empty and set the flag; the
    other requests of the same warp task (per-lane FSM path) still match."""
    d = configs.config2(n=100, gid0=4242)
    data, off = d["data"], d["offsets"].copy()
    off[37] = off[39]  # request 36 = [off36, off39) overlaps 37; request 37 = [off39, off38) has e < s
    ctx_v1.flags()  # clear
    feat = ctx_v1.score(dev(data), dev(off))
    torch.cuda.synchronize()
    got = host(feat, np.uint16)
    assert ctx_v1.flags() & 2
    for i in range(100):
        s, e = int(off[i]), int(off[i + 1])
        if e < s:
            assert (got[i] == 0).all()
            continue
        seg = np.ascontiguousarray(data[s:e])
        want = oracle.rule_gen(lex_v1, seg, np.asarray([0, e - s], np.uint32))
        assert (got[i] == want[0]).all(), i


@pytest.mark.parametrize("ratio", [0.0, 0.3, 1.0])
def test_malicious_workload(ctx_v1, lex_v1, ratio):
    """NEXT-3: the malicious-task sweep reuses K1-K6 unchanged:
    scoring of the crafted texts and the replay match the oracle."""
    d = configs.with_malicious(configs.traces(3, range(200, 216), 1000, lambda t: t % 4), ratio)
    feat = ctx_v1.score(dev(d["data"]), dev(d["offsets"]))
    torch.cuda.synchronize()
    f = oracle.rule_gen(lex_v1, d["data"], d["offsets"])
    assert (host(feat, np.uint16) == f).all()
    for ov in ({}, {"policy": "FIFO", "consolidate": 0, "offload": 0}):
        _replay_case(ctx_v1, lex_v1, d, ov)


@pytest.mark.parametrize("policy_ov", [{}, {"consolidate": 0}, {"offload": 0, "cores": 1}])
def test_replay_rank_ties_and_ragged_traces(ctx_v1, policy_ov):
    """k_trace_rank + k_replay on ragged traces (1 .. 1024 tasks, non-powers of
    two) whose keys and u take only a few distinct values: the priority order
    is then decided by the arrival-index tie-break (R-TIE) and the window's
    (u, rank) order by the rank; end times against the oracle."""
    rng = np.random.default_rng(11)
    sizes = [1, 2, 3, 31, 32, 33, 63, 500, 1000, 1023, 1024, 7]
    toff = np.concatenate([[0], np.cumsum(sizes)]).astype(U32)
    n = int(toff[-1])
    arr = np.concatenate([np.sort(rng.integers(0, 30_000_000, s)) for s in sizes]).astype(np.int64)
    arr[toff[3]:toff[4]] = 5_000_000  # a trace whose tasks all arrive together
    low = rng.choice(np.asarray([3, 3, 7, 1 << 40], np.uint64), n)
    cls = (rng.random(n) < 0.2).astype(np.uint64) << np.uint64(63)
    key = (cls | low).astype(np.uint64)
    u = rng.choice(np.asarray([5.0, 5.0, 12.5, 40.0], np.float32), n)
    tl = rng.integers(1, 80, n).astype(np.uint16)
    D = rng.integers(1_000_000, 20_000_000, n).astype(U32)
    profs = [dict(p, **policy_ov) for p in configs.paper_lms()]
    tp = (np.arange(len(sizes)) % 4).astype(np.uint16)
    st, end = oracle.simulate(arr, tl, u, key, D, toff, profs, tp, want_end=True)
    gs, gend = ctx_v1.simulate(dev(arr), dev(tl), dev(u), dev(key), dev(D), toff, profs, dev(tp), want_end=True)
    torch.cuda.synchronize()
    assert (rt.decode_stats(gs) == st).all()
    assert (gend.cpu().numpy() == end).all()


def test_score_schedule_host_matches_oracle(ctx_v1, lex_v1):
    """rt_score_schedule_host (the e2e entry: host buffers in, host assignment
    out) equals the oracle's one-pass schedule on a config-2 prefix queue."""
    d = configs.config2(n=20000)
    n = len(d["offsets"]) - 1
    hb = torch.from_numpy(d["data"]).pin_memory()
    ho = torch.from_numpy(d["offsets"].view(np.int32)).pin_memory()
    out = {"batch_of": torch.empty(n, dtype=torch.int32).pin_memory(),
           "slot_of": torch.empty(n, dtype=torch.uint8).pin_memory(),
           "core_of": torch.empty(n, dtype=torch.uint8).pin_memory()}
    ctx_v1.score_schedule_host(hb, ho, d["regressor"], d["profile"], out)
    torch.cuda.synchronize()
    f = oracle.rule_gen(lex_v1, d["data"], d["offsets"])
    u = oracle.predict(f, d["regressor"])
    k, _ = oracle.key(u, f, d["profile"])
    s = oracle.schedule(k, u, np.asarray([0, n], U32), d["profile"])
    assert (out["batch_of"].numpy().view(U32) == s["batch_of"]).all()
    assert (out["slot_of"].numpy() == s["slot_of"]).all()
    assert (out["core_of"].numpy() == s["core_of"]).all()


def test_graph_capture_of_the_step(ctx_v1, lex_v1):
    """rt_score_key + rt_schedule captured in a CUDA graph (the bench's pipelined
    step) and replayed: bit-identical to the call-by-call path; staged host
    offsets of the capture stay valid after later normal calls."""
    d = configs.config2(n=30000)
    n = len(d["offsets"]) - 1
    data, off = dev(d["data"]), dev(d["offsets"])
    seg = np.asarray([0, n], U32)
    o1 = ctx_v1.score_key(data, off, d["regressor"], d["profile"], want_D=False)
    s1 = ctx_v1.schedule(o1["key"], o1["u"], seg, d["profile"])
    ref = {k: v.clone() for k, v in s1.items()}
    torch.cuda.synchronize()
    st = torch.cuda.Stream(DEV)
    outs = {"u": torch.empty(n, dtype=torch.float32, device=DEV), "key": torch.empty(n, dtype=torch.int64, device=DEV)}
    souts = {k: torch.empty_like(v) for k, v in ref.items()}
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
        ctx_v1.score_key(data, off, d["regressor"], d["profile"], want_D=False, out=outs)
        ctx_v1.schedule(outs["key"], outs["u"], seg, d["profile"], out=souts)
    for k in souts:
        souts[k].zero_()
    # a normal call on another queue size in between (re-stages offsets)
    o2 = ctx_v1.score_key(data, off, d["regressor"], d["profile"], want_D=False)
    ctx_v1.schedule(o2["key"], o2["u"], np.asarray([0, 100, n], U32), d["profile"])
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    for k in ref:
        assert torch.equal(souts[k], ref[k]), k


@pytest.mark.parametrize("policy", ["UP", "EDF", "FIFO"])
def test_schedule_deadlines_form(ctx_v1, lex_v1, policy):
    """rt_schedule_deadlines (north-star form: queue, deadlines, cores): keys from
    u and caller deadlines in-call; equals the oracle's key + schedule on several
    queues (one big, two small), arrivals given for FIFO/EDF."""
    d = configs.config2(n=6000)
    prof = dict(d["profile"], policy=policy)
    n = len(d["offsets"]) - 1
    rng = np.random.default_rng(5)
    f = oracle.rule_gen(lex_v1, d["data"], d["offsets"])
    u = oracle.predict(f, d["regressor"])
    D = rng.integers(1, 3_000_000, n).astype(U32)
    arr = np.sort(rng.integers(0, 10_000_000, n)).astype(np.int64)
    k, _ = oracle.key(u, f, prof, r_us=arr, D_in=D)
    seg = np.asarray([0, 100, 2148, n], U32)
    s = oracle.schedule(k, u, seg, prof)
    g = ctx_v1.schedule_deadlines(dev(u), dev(D), seg, prof, arrival=dev(arr))
    torch.cuda.synchronize()
    _check_schedule(g, s, 3)


@pytest.mark.parametrize("tight", [1, 2])
@pytest.mark.parametrize("ov", [{}, {"policy": "EDF", "consolidate": 0, "offload": 0}, {"policy": "LUF", "consolidate": 0,
                                                                                        "offload": 0}])
def test_periodic_release_replay(ctx_v1, lex_v1, tight, ov):
    """NEXT-3 periodic scenario: each task is released at the
    previous task's deadline, tight (mu*|J|) or loose (twice).  Deadlines and
    keys from the GPU path, arrivals from them, replay; all against the oracle
    (the oracle computes its own deadlines and keys from the same features)."""
    d = configs.traces(3, range(300, 308), 400, lambda t: t % 4)
    profs = [dict(p, tightness=tight, **ov) for p in d["profiles"]]
    n = len(d["true_len"])
    f = oracle.rule_gen(lex_v1, d["data"], d["offsets"])
    u = np.zeros(n, np.float32)
    D = np.zeros(n, U32)
    for t in range(len(d["trace_off"]) - 1):
        lo, hi = int(d["trace_off"][t]), int(d["trace_off"][t + 1])
        lm = int(d["trace_prof"][t])
        u[lo:hi] = oracle.predict(f[lo:hi], d["regressors"][lm])
        _, D[lo:hi] = oracle.key(u[lo:hi], f[lo:hi], profs[lm])
    arr = configs.periodic_arrivals(d["trace_off"], D)
    k = np.zeros(n, np.uint64)
    for t in range(len(d["trace_off"]) - 1):
        lo, hi = int(d["trace_off"][t]), int(d["trace_off"][t + 1])
        k[lo:hi], _ = oracle.key(u[lo:hi], f[lo:hi], profs[int(d["trace_prof"][t])], r_us=arr[lo:hi])
    st, end = oracle.simulate(arr, d["true_len"], u, k, D, d["trace_off"], profs, d["trace_prof"], want_end=True)
    # GPU: keys from the device path with the periodic arrivals, then the replay
    gk = torch.empty(n, dtype=torch.int64, device=DEV)
    gD = torch.empty(n, dtype=torch.int32, device=DEV)
    gfeat, gu, garr = dev(f), dev(u), dev(arr)
    for t in range(len(d["trace_off"]) - 1):
        lo, hi = int(d["trace_off"][t]), int(d["trace_off"][t + 1])
        ctx_v1.key(gu[lo:hi], profs[int(d["trace_prof"][t])], feat=gfeat[lo:hi], arrival=garr[lo:hi], key=gk[lo:hi],
                   D_out=gD[lo:hi])
    gs, gend = ctx_v1.simulate(garr, dev(d["true_len"]), gu, gk, gD, d["trace_off"], profs, dev(d["trace_prof"]),
                               want_end=True)
    torch.cuda.synchronize()
    assert (gD.cpu().numpy().view(U32) == D).all()
    assert (rt.decode_stats(gs) == st).all()
    assert (gend.cpu().numpy() == end).all()


@pytest.mark.parametrize("which", ["small", "medium", "large"])
def test_variance_subset_traces(ctx_v1, lex_v1, which):
    """NEXT-3 variance subsets: tasks gathered from a scored pool by the
    spread of u, packed into Poisson traces; keys and replay on the GPU against
    the oracle (FIFO / LUF / MUF without consolidation, UP+C+O)."""
    pool = configs.traces(3, range(500, 504), 1000, lambda t: 0)
    f = oracle.rule_gen(lex_v1, pool["data"], pool["offsets"])
    u = oracle.predict(f, pool["regressors"][0])
    idx = configs.variance_subsets(u, 1200)[which]
    per, nt = 400, 3
    toff = (np.arange(nt + 1) * per).astype(U32)
    arr = np.concatenate([rtgen.arrivals(rtgen.ROOT_SEED + 3, 700 + t, per) for t in range(nt)])
    fs, us, tl = f[idx], u[idx], pool["true_len"][idx]
    tp = np.zeros(nt, np.uint16)
    for ov in ({"policy": "FIFO", "consolidate": 0, "offload": 0}, {"policy": "LUF", "consolidate": 0, "offload": 0},
               {"policy": "MUF", "consolidate": 0, "offload": 0}, {}):
        prof = dict(pool["profiles"][0], **ov)
        k, D = oracle.key(us, fs, prof, r_us=arr)
        st, end = oracle.simulate(arr, tl, us, k, D, toff, [prof], tp, want_end=True)
        gk, gD = ctx_v1.key(dev(us), prof, feat=dev(fs), arrival=dev(arr))
        gs, gend = ctx_v1.simulate(dev(arr), dev(tl), dev(us), gk, gD, toff, [prof], dev(tp), want_end=True)
        torch.cuda.synchronize()
        assert (host(gk, np.uint64) == k).all()
        assert (rt.decode_stats(gs) == st).all()
        assert (gend.cpu().numpy() == end).all()
