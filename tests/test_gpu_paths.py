"""GPU parity of the launch configurations and kernel paths the round-1 tests did
not reach ("Next round" item 2):

* the bench's timed requests step exactly as bench.py runs it: `depth` = 4
  batches in flight, one context + stream + distinct 2^20-request input per
  batch, the persistent scoring kernel capped by rt_set_sm_limit(nsm - 4),
  issued call by call and replayed from CUDA graphs -- every batch's order,
  batches, slots and cores against the oracle;
* crafted-u big queues (> 2048, the parallel consolidation path of k_ff.cu):
  the exact fp32 lambda boundary (u == fl(lambda * u_prev), and one ulp above),
  runs of u = 0, all-equal streams, u monotone along the priority order;
* the CPU-class list-scheduling chain on 4 cores in all three arithmetic
  forms of k_cpu_chain (u32 offsets from a base, u32 deltas, u64 keys), which
  only predicted CPU latencies above ~119 s reach (u >~ 475 tokens at
  DialoGPT's gamma and eta);
* a 1024-entry lexicon (the cap) of 12-16-byte lemmas, with near misses in
  bytes 13-16, inflected and clitic forms;
* argument checks that must launch nothing (rtlm.h: argument checks are
  synchronous and launch nothing), including offload with zero cores.
"""
import zlib

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


def check_schedule(g, s, nq):
    assert (host(g["perm"], U32) == s["perm"]).all(), "perm"
    assert (host(g["batch_of"], U32) == s["batch_of"]).all(), "batch_of"
    assert (g["slot_of"].cpu().numpy() == s["slot_of"]).all(), "slot_of"
    assert (g["core_of"].cpu().numpy() == s["core_of"]).all(), "core_of"
    assert (host(g["seg_batch_off"], U32)[:nq + 1] == s["seg_batch_off"]).all(), "seg_batch_off"


@pytest.fixture(scope="module")
def ctx_v1():
    return rt.Context(configs.read_lexicon(), 0)


# ------------------------------------------------------------------ the bench's timed step
@pytest.mark.parametrize("mode", ["split", "slot", "graphs"])
def test_bench_pipeline_launch_configuration(lex_v1, mode):
    """bench.py's pipelined requests leg in each of its launch forms: "split"
    (the default: every batch's scoring on one stream with the persistent
    kernel capped at ~2/3 of the SMs, each batch's schedule on its slot's stream,
    ordered by events; depth 8), "slot" (score + schedule on the slot's stream,
    scoring capped at nsm - depth; depth 4) and "graphs" (slot form, each slot's
    step replayed from one CUDA graph).  Two waves of steps so that every slot
    runs while other slots' kernels are in flight; every batch against the oracle."""
    n = 1 << 20
    depth = 8 if mode == "split" else 4
    steps = 2 * depth
    nsm = torch.cuda.get_device_properties(DEV).multi_processor_count
    ds = [configs.config2(n=n, gid0=i * n) for i in range(depth)]
    prof, reg = ds[0]["profile"], ds[0]["regressor"]
    seg = np.asarray([0, n], U32)
    ctxs = [rt.Context(d["lexicon"], 0) for d in ds]
    for c in ctxs:
        c.set_sm_limit((nsm * 100 + 74) // 148 if mode == "split" else max(1, nsm - depth))
    data = [dev(d["data"]) for d in ds]
    off = [dev(d["offsets"]) for d in ds]
    streams = [torch.cuda.Stream(DEV) for _ in range(depth)]
    score_stream = torch.cuda.Stream(DEV)
    ev_scored = [torch.cuda.Event() for _ in range(depth)]
    ev_sched = [torch.cuda.Event() for _ in range(depth)]
    outs = [{"u": torch.empty(n, dtype=torch.float32, device=DEV), "key": torch.empty(n, dtype=torch.int64, device=DEV)}
            for _ in range(depth)]
    souts = [{"perm": torch.empty(n, dtype=torch.int32, device=DEV),
              "batch_of": torch.empty(n, dtype=torch.int32, device=DEV),
              "slot_of": torch.empty(n, dtype=torch.uint8, device=DEV),
              "core_of": torch.empty(n, dtype=torch.uint8, device=DEV),
              "seg_batch_off": torch.empty(2, dtype=torch.int32, device=DEV)} for _ in range(depth)]

    def pstep(k):
        sl = k % depth
        if mode == "split":
            with torch.cuda.stream(score_stream):
                score_stream.wait_event(ev_sched[sl])
                ctxs[sl].score_key(data[sl], off[sl], reg, prof, want_D=False, out=outs[sl])
                ev_scored[sl].record(score_stream)
            with torch.cuda.stream(streams[sl]):
                streams[sl].wait_event(ev_scored[sl])
                ctxs[sl].schedule(outs[sl]["key"], outs[sl]["u"], seg, prof, out=souts[sl])
                ev_sched[sl].record(streams[sl])
            return
        with torch.cuda.stream(streams[sl]):
            ctxs[sl].score_key(data[sl], off[sl], reg, prof, want_D=False, out=outs[sl])
            ctxs[sl].schedule(outs[sl]["key"], outs[sl]["u"], seg, prof, out=souts[sl])

    for k in range(depth):  # warm-up: every slot runs before its capture
        pstep(k)
    torch.cuda.synchronize()
    for o in souts:  # poison the outputs: the waves below must rewrite them
        for t in o.values():
            t.fill_(-1 if t.dtype != torch.uint8 else 0x7F)
    torch.cuda.synchronize()
    if mode == "graphs":
        gs = []
        for sl in range(depth):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=streams[sl], capture_error_mode="relaxed"):
                pstep(sl)
            gs.append(g)
        torch.cuda.synchronize()
        for k in range(steps):
            with torch.cuda.stream(streams[k % depth]):
                gs[k % depth].replay()
    else:
        for k in range(steps):
            pstep(k)
    torch.cuda.synchronize()
    for c in ctxs:
        c.set_sm_limit(0)
    for sl, d in enumerate(ds):
        f = oracle.rule_gen(lex_v1, d["data"], d["offsets"])
        u = oracle.predict(f, reg)
        k, _ = oracle.key(u, f, prof)
        assert (host(outs[sl]["key"], np.uint64) == k).all(), f"slot {sl}: keys"
        assert (outs[sl]["u"].cpu().numpy().view(U32) == u.view(U32)).all(), f"slot {sl}: u"
        check_schedule(souts[sl], oracle.schedule(k, u, seg, prof), 1)


# ------------------------------------------------------------------ crafted-u big queues
def crafted_u(kind: str, n: int, rng) -> np.ndarray:
    if kind == "lambda_boundary":
        # u_{j+1} = fl(1.5 * u_j) exactly (8 * 1.5^j is exact in binary32 for j < 20),
        # the next binary32 above it, and a few random values
        geo = (8.0 * 1.5 ** np.arange(12)).astype(np.float32)
        above = np.nextafter(geo, np.float32(np.inf)).astype(np.float32)
        below = np.nextafter(geo, np.float32(0)).astype(np.float32)
        pool = np.concatenate([geo, geo, geo, above, below, rng.uniform(1, 600, 8).astype(np.float32)])
        return rng.choice(pool, n).astype(np.float32)
    if kind == "zero_runs":
        u = rng.uniform(0.5, 30, n).astype(np.float32)
        i = 0
        while i < n:  # runs of zeros of random length
            L = int(rng.integers(1, 200))
            if rng.random() < 0.5:
                u[i:i + L] = 0.0
            i += L + int(rng.integers(1, 100))
        return u
    if kind == "all_equal":
        return np.full(n, 7.25, np.float32)
    if kind in ("monotone_up", "monotone_down"):
        return rng.uniform(0.0, 600.0, n).astype(np.float32)
    raise ValueError(kind)


@pytest.mark.parametrize("n", [3001, 40000])
@pytest.mark.parametrize("kind", ["lambda_boundary", "zero_runs", "all_equal", "monotone_up", "monotone_down"])
@pytest.mark.parametrize("lam,C,b10", [(1.5, 11, 18), (1.5, 33, 30), (1.0, 8, 10)])
def test_schedule_crafted_u(ctx_v1, kind, n, lam, C, b10):
    rng = np.random.default_rng(zlib.crc32(f"{kind}/{n}/{lam}/{C}".encode()))
    u = crafted_u(kind, n, rng)
    # monotone along the priority order: LUF serves ascending u, MUF descending u
    policy = {"monotone_up": "LUF", "monotone_down": "MUF"}.get(kind, "UP")
    prof = dict(configs.paper_lms()[0], policy=policy, offload=0, C=C, b10=b10, **{"lambda": lam})
    D = rng.integers(1, 3_000_000, n).astype(U32)
    f = np.zeros((n, 8), np.uint16)
    k, _ = oracle.key(u, f, prof, D_in=D)
    seg = np.asarray([0, n], U32)
    s = oracle.schedule(k, u, seg, prof)
    g = ctx_v1.schedule_deadlines(dev(u), dev(D), seg, prof)
    torch.cuda.synchronize()
    check_schedule(g, s, 1)
    if kind == "lambda_boundary" and lam == 1.5:
        # the boundary is really exercised: some batch holds a pair (x, fl(1.5 x)) adjacent in u order
        bo, uu = s["batch_of"], u
        hit = False
        for b in np.unique(bo)[:2000]:
            m = np.sort(uu[bo == b])
            if len(m) > 1 and np.any(m[1:] == (np.float32(1.5) * m[:-1]).astype(np.float32)) and np.any(m[1:] != m[:-1]):
                hit = True
                break
        assert hit


def test_cpu_chain_arithmetic_forms(ctx_v1):
    """k_cpu_chain on 4 cores: the CPU class in ascending-u order (LUF) passes from
    small predicted latencies (u32 offsets from a base), through 119-134 s (u32
    deltas: u in [475, 536]), to latencies above 2^27 us (u64 keys)."""
    n = 60000
    rng = np.random.default_rng(2024)
    prof = dict(configs.paper_lms()[0], policy="LUF", offload=1, cores=4)
    gpu = rng.uniform(0.0, 35.0, 24000)
    bands = [rng.uniform(35.5, 400.0, 12000), rng.uniform(480.0, 530.0, 12000), rng.uniform(600.0, 2.0e5, 12000)]
    u = np.concatenate([gpu] + bands).astype(np.float32)
    rng.shuffle(u)
    D = rng.integers(1, 3_000_000, n).astype(U32)
    f = np.zeros((n, 8), np.uint16)
    k, _ = oracle.key(u, f, prof, D_in=D)
    seg = np.asarray([0, n], U32)
    eta, gam, base = np.float32(prof["eta_us"]), prof["gamma"], prof["base_us"]
    pred = gam * (base + np.ceil((eta * u).astype(np.float32)).astype(np.int64))
    assert pred.max() >= 1 << 27 and ((pred >= 119_000_000) & (pred < 1 << 27)).sum() > 4096
    s = oracle.schedule(k, u, seg, prof)
    g = ctx_v1.schedule_deadlines(dev(u), dev(D), seg, prof)
    torch.cuda.synchronize()
    check_schedule(g, s, 1)


# ------------------------------------------------------------------ 1024-entry lexicon
def long_lexicon(rng):
    """1024 distinct lemmas of 12-16 letters that the loader's lemmatizer leaves
    unchanged (no final s / ed / ing), spread over every section."""
    alpha = np.frombuffer(b"abcdefghijklmnopqrtuvwxyz", np.uint8)  # no 's'
    words = set()
    while len(words) < 1024:
        L = int(rng.integers(12, 17))
        w = bytes(rng.choice(alpha, L)).decode()
        if w.endswith(("ed", "ing", "s")):
            continue
        words.add(w)
    words = sorted(words)
    rng.shuffle(words)
    sec = {"vague": words[0:200], "polysemy": words[200:400], "pos": words[400:700], "wh": words[700:820],
           "coord": words[820:900], "prep": words[900:1024]}
    lines = ["vague:"] + sec["vague"]
    lines += ["polysemy:"] + [f"{w}\t{int(rng.integers(2, 9))}" for w in sec["polysemy"]]
    tags = ["NOUN", "PROPN", "VERB", "ADJ", "NOUN,VERB", "VERB,ADP", "NOUN,ADJ"]
    lines += ["pos:"] + [f"{w}\t{tags[int(rng.integers(0, len(tags)))]}" for w in sec["pos"]]
    flags = ["OPENER", "WHAT", "CAUSE", "BROAD", "OPENER|BROAD", "WHAT|CAUSE"]
    lines += ["wh:"] + [f"{w}\t{flags[int(rng.integers(0, len(flags)))]}" for w in sec["wh"]]
    lines += ["coord:"] + sec["coord"] + ["prep:"] + sec["prep"]
    return "\n".join(lines) + "\n", words


def near_miss_texts(words, rng):
    out = []
    for _ in range(3000):
        toks = []
        for _ in range(int(rng.integers(1, 30))):
            w = words[int(rng.integers(0, len(words)))]
            r = rng.random()
            if r < 0.3:
                pass                                                     # exact hit
            elif r < 0.5 and len(w) >= 13:                               # near miss in bytes 13..16
                j = int(rng.integers(12, len(w)))
                w = w[:j] + ("z" if w[j] != "z" else "y") + w[j + 1:]
            elif r < 0.6:
                w = w + "x"                                              # 13..17 bytes: extension
            elif r < 0.65:
                w = w[:-1]                                               # truncation
            elif r < 0.75:
                w = w + ["s", "ed", "ing", "es"][int(rng.integers(0, 4))]  # inflections -> lemma (R-LEMMA)
            elif r < 0.85:
                w = w + ["'s", "n't", "'ll", "'re", "'d"][int(rng.integers(0, 5))]  # clitics (R-CLITIC)
            elif r < 0.92:
                w = w.upper()
            else:
                w = ["?", ",", ".", "!", "and", "the"][int(rng.integers(0, 6))]
            toks.append(w)
        out.append(" ".join(toks))
    return out


def test_lexicon_1024_long_lemmas():
    rng = np.random.default_rng(1024)
    text, words = long_lexicon(rng)
    lex = oracle.Lexicon(text)
    assert len(lex) == 1024
    ctx = rt.Context(text, 0)
    assert ctx.lexicon_size == 1024
    data, off = rtgen.pack_texts(near_miss_texts(words, rng))
    feat = ctx.score(dev(data), dev(off))
    torch.cuda.synchronize()
    got, want = host(feat, np.uint16), oracle.rule_gen(lex, data, off)
    bad = np.nonzero((got != want).any(1))[0]
    assert len(bad) == 0, [(int(i), got[i].tolist(), want[i].tolist()) for i in bad[:5]]
    assert (want[:, 3] > 0).mean() > 0.3 and (want[:, 2] > 0).mean() > 0.3  # V and M really fire
    # one more distinct lemma than the cap is a lexicon error
    with pytest.raises(rt.RtlmError, match="more than 1024"):
        rt.Context(text + "vague:\nqqqqqqqqqqqqqq\n", 0)


def test_senses_saturation_in_the_pool_path():
    """M (sum of senses - 1) saturates at 65535 and sets RT_FLAG_SATURATED for a
    request small enough for the pool path (not the byte FSM): 300 words of 255
    senses = 76 200; its neighbours in the same warp task stay exact."""
    text = "polysemy:\nbat\t255\nbank\t3\n"
    lex = oracle.Lexicon(text)
    ctx = rt.Context(text, 0)
    t = ["bat " * 300, "bats and banks", "bat " * 257 + "bank", "bat " * 259, ""] + ["bank bat"] * 40
    data, off = rtgen.pack_texts(t)
    ctx.flags()
    feat = ctx.score(dev(data), dev(off))
    torch.cuda.synchronize()
    got, want = host(feat, np.uint16), oracle.rule_gen(lex, data, off)
    assert (got == want).all(), [(i, got[i].tolist(), want[i].tolist()) for i in np.nonzero((got != want).any(1))[0][:5]]
    assert want[0, 2] == 65535 and want[2, 2] == 257 * 254 + 2 and want[3, 2] == 65535
    assert ctx.flags() & 1


@pytest.mark.parametrize("order", [0, 1])
def test_lexicon_fingerprint_collision(order):
    """The probe compares only the key whose slot fingerprint matches; when both
    slots' fingerprints match and the first key differs it compares the second.
    "dvpczvzzu" and "wnhunduzd" share a 21-bit fingerprint and their first slot
    (seed 0, 64 slots; found by a search over the library's published hash,
    lex_mix / lex_slot1 in csrc/internal.cuh): the word inserted second sits in
    its second slot, behind the other word's matching fingerprint."""
    a, b = "dvpczvzzu", "wnhunduzd"
    first, second = (b, a) if order == 0 else (a, b)
    text = f"vague:\n{first}\npolysemy:\n{second}\t3\n"
    lex = oracle.Lexicon(text)
    ctx = rt.Context(text, 0)
    t = [f"{second}", f"{first}", f"{second} {first} {second.upper()}", f"{second}s and {first}'s", "other"] * 8
    data, off = rtgen.pack_texts(t)
    feat = ctx.score(dev(data), dev(off))
    torch.cuda.synchronize()
    got, want = host(feat, np.uint16), oracle.rule_gen(lex, data, off)
    assert (got == want).all(), [(i, got[i].tolist(), want[i].tolist()) for i in np.nonzero((got != want).any(1))[0][:5]]
    assert want[1, 3] == 1 and want[0, 2] == 2 and want[2, 2] == 4  # the first word VAGUE, the second 3 senses


# ------------------------------------------------------------------ argument checks launch nothing
def test_schedule_argument_checks_launch_nothing(ctx_v1):
    n = 5000
    u = torch.ones(n, dtype=torch.float32, device=DEV)
    D = torch.full((n,), 1000, dtype=torch.int32, device=DEV)
    key = torch.zeros(n, dtype=torch.int64, device=DEV)
    p = dict(configs.paper_lms()[0])
    torch.cuda.synchronize()
    l0 = rt.launch_count()
    with pytest.raises(rt.RtlmError, match="cores"):
        ctx_v1.schedule(key, u, np.asarray([0, n], U32), dict(p, offload=1), cores=0)
    with pytest.raises(rt.RtlmError, match="cores"):
        ctx_v1.schedule_deadlines(u, D, np.asarray([0, n], U32), dict(p, offload=1), cores=0)
    with pytest.raises(rt.RtlmError, match="non-decreasing"):
        ctx_v1.schedule_deadlines(u, D, np.asarray([0, 3000, 2000, n], U32), p)
    with pytest.raises(rt.RtlmError, match="lambda"):
        ctx_v1.schedule_deadlines(u, D, np.asarray([0, n], U32), dict(p, **{"lambda": 0.5}))
    h = torch.from_numpy(np.zeros(64, np.uint8))
    ho = torch.from_numpy(np.asarray([0, 32, 64], np.int32))
    res = {"batch_of": torch.empty(2, dtype=torch.int32), "slot_of": torch.empty(2, dtype=torch.uint8),
           "core_of": torch.empty(2, dtype=torch.uint8)}
    with pytest.raises(rt.RtlmError, match="cores"):
        ctx_v1.score_schedule_host(h, ho, configs.regressor(p), dict(p, offload=1, cores=0), res)
    assert rt.launch_count() == l0, "a rejected call launched kernels"
    # without offload, zero cores is valid (no CPU class)
    g = ctx_v1.schedule(key, u, np.asarray([0, n], U32), dict(p, offload=0), cores=0)
    torch.cuda.synchronize()
    assert (g["core_of"].cpu().numpy() == 0xFF).all()


# ------------------------------------------------------------------ long traces (k_replay_long)
def _replay_vs_oracle(ctx, arr, tl, u, key, D, toff, profs, tp):
    st, end = oracle.simulate(arr, tl, u, key, D, toff, profs, tp, want_end=True)
    gs, gend = ctx.simulate(dev(arr), dev(tl), dev(u), dev(key), dev(D), toff, profs, dev(tp), want_end=True)
    torch.cuda.synchronize()
    g = rt.decode_stats(gs)
    assert (g == st).all(), [(i, g[i], st[i]) for i in np.nonzero(g != st)[0][:3]]
    assert (gend.cpu().numpy() == end).all()
    return st


@pytest.mark.parametrize("ov", [{}, {"consolidate": 0}, {"offload": 0}, {"policy": "EDF"}, {"tightness": 2},
                                {"policy": "FIFO", "consolidate": 0, "offload": 0}])
def test_replay_full_paper_ramp(ctx_v1, lex_v1, ov):
    """Whole traces of the paper's workload: beta = 10, 11, .., 150 arrivals per
    minute, one minute each = 11 280 Poisson arrivals per trace,
    beside ordinary 1000-task traces in the same call; end times and stats
    exact against the oracle."""
    d = configs.traces(3, range(900, 904), 11280, lambda t: t % 4)
    assert d["arrival_us"][11279] > 130 * 60_000_000  # the ramp really spans ~141 minutes
    short = configs.traces(3, range(950, 953), 1000, lambda t: (t + 1) % 4)
    cat = {k: np.concatenate([d[k], short[k]]) for k in ("arrival_us", "true_len", "trace_prof")}
    toff = np.concatenate([d["trace_off"], d["trace_off"][-1] + short["trace_off"][1:]]).astype(U32)
    profs = [dict(p, **ov) for p in d["profiles"]]
    u, k, D = [], [], []
    for dd in (d, short):
        f = oracle.rule_gen(lex_v1, dd["data"], dd["offsets"])
        for t in range(len(dd["trace_off"]) - 1):
            lo, hi = int(dd["trace_off"][t]), int(dd["trace_off"][t + 1])
            lm = int(dd["trace_prof"][t])
            ut = oracle.predict(f[lo:hi], dd["regressors"][lm])
            kt, Dt = oracle.key(ut, f[lo:hi], profs[lm], r_us=dd["arrival_us"][lo:hi])
            u.append(ut), k.append(kt), D.append(Dt)
    st = _replay_vs_oracle(ctx_v1, cat["arrival_us"], cat["true_len"], np.concatenate(u), np.concatenate(k),
                           np.concatenate(D), toff, profs, cat["trace_prof"])
    assert st["n"][0] == 11280 and st["n"][-1] == 1000


@pytest.mark.parametrize("policy_ov", [{}, {"consolidate": 0}, {"offload": 0, "cores": 1}, {"b10": 30, "C": 33}])
def test_replay_long_ties_and_sizes(ctx_v1, policy_ov):
    """k_replay_long on traces of 1025 .. 65536 tasks with few distinct keys and u
    values (rank ties broken by arrival index, R-TIE), bursts arriving together,
    and an overload that keeps thousands of tasks ready."""
    rng = np.random.default_rng(77)
    sizes = [1025, 2048, 3001, 1024, 17, 65536]
    toff = np.concatenate([[0], np.cumsum(sizes)]).astype(U32)
    n = int(toff[-1])
    arr = np.concatenate([np.sort(rng.integers(0, 20_000_000 * max(1, s // 1000), s)) for s in sizes]).astype(np.int64)
    arr[toff[1]:toff[1] + 700] = arr[toff[1]]  # a burst of 700 simultaneous arrivals
    arr[toff[1]:toff[2]] = np.sort(arr[toff[1]:toff[2]])
    low = rng.choice(np.asarray([3, 3, 7, 1 << 40], np.uint64), n)
    cls = (rng.random(n) < 0.2).astype(np.uint64) << np.uint64(63)
    key = (cls | low).astype(np.uint64)
    u = rng.choice(np.asarray([5.0, 5.0, 12.5, 40.0], np.float32), n)
    tl = rng.integers(1, 80, n).astype(np.uint16)
    D = rng.integers(1_000_000, 20_000_000, n).astype(U32)
    profs = [dict(p, **policy_ov) for p in configs.paper_lms()]
    tp = (np.arange(len(sizes)) % 4).astype(np.uint16)
    _replay_vs_oracle(ctx_v1, arr, tl, u, key, D, toff, profs, tp)


def test_replay_rejects_traces_over_65536(ctx_v1):
    n = 65537
    z = torch.zeros(n, dtype=torch.int64, device=DEV)
    with pytest.raises(rt.RtlmError, match="65536"):
        ctx_v1.simulate(z, torch.zeros(n, dtype=torch.int16, device=DEV), torch.zeros(n, device=DEV), z,
                        torch.zeros(n, dtype=torch.int32, device=DEV), np.asarray([0, n], U32),
                        [configs.paper_lms()[0]], None)


def test_config4_two_streams_match_one():
    """bench.py's config-4 step: blocks alternate between two contexts and
    streams (scoring capped at half the SMs), stats accumulated by both with
    atomics.  Per-trace stats and per-LM sums equal the one-context serial run."""
    from bench import _lm_groups
    blocks = []
    for blk in range(4):
        d = configs.config4_shard(blk, 4, n_traces=512, per_trace=256, grouped=True)
        blocks.append({"d": d, "groups": _lm_groups(d, DEV), "arr": dev(d["arrival_us"]), "tl": dev(d["true_len"]),
                       "tp": dev(d["trace_prof"])})
    lex = blocks[0]["d"]["lexicon"]
    ctxs = [rt.Context(lex, 0), rt.Context(lex, 0)]
    nsm = torch.cuda.get_device_properties(DEV).multi_processor_count

    def run(nstreams):
        streams = [torch.cuda.Stream(DEV) for _ in range(nstreams)]
        for c in ctxs:
            c.set_sm_limit((nsm + 1) // 2 if nstreams > 1 else 0)
        sums = torch.zeros((4, 3), dtype=torch.int64, device=DEV)
        ev0 = torch.cuda.Event()
        ev0.record()
        stats = []
        for i, b in enumerate(blocks):
            c, st = ctxs[i % nstreams], streams[i % nstreams]
            d, arr = b["d"], b["arr"]
            nb, ntb = len(d["arrival_us"]), len(d["trace_off"]) - 1
            with torch.cuda.stream(st):
                if i < nstreams:
                    st.wait_event(ev0)
                u = torch.empty(nb, dtype=torch.float32, device=DEV)
                key = torch.empty(nb, dtype=torch.int64, device=DEV)
                D = torch.empty(nb, dtype=torch.int32, device=DEV)
                s = torch.empty((ntb, 2), dtype=torch.int64, device=DEV)
                for f, r0, r1, gd, so in b["groups"]:
                    c.score_key(gd, so, d["regressors"][f], d["profiles"][f], arrival=arr[r0:r1],
                                out={"u": u[r0:r1], "key": key[r0:r1], "D": D[r0:r1]})
                c.simulate(arr, b["tl"], u, key, D, d["trace_off"], d["profiles"], b["tp"], stats=s)
                c.reduce_stats(s, b["tp"], 4, sums=sums)
                stats.append(s)
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
        torch.cuda.synchronize()
        for c in ctxs:
            c.set_sm_limit(0)
        return [s.cpu().numpy() for s in stats], sums.cpu().numpy()

    st1, s1 = run(1)
    st2, s2 = run(2)
    for a, b in zip(st1, st2):
        assert (a == b).all()
    assert (s1 == s2).all()
    assert s1[:, 1].sum() == sum(len(b["d"]["arrival_us"]) for b in blocks)  # every request counted once
