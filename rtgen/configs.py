"""Concrete workloads of BASELINE.json's five configs, built
from rtgen only.  Harness code: no method arithmetic (no features, no keys).

Every function returns plain numpy arrays plus profile dicts taken from
data/profiles.json (written by scripts/calibrate.py).
"""
from __future__ import annotations

import json
import os

import numpy as np

from . import ROOT_SEED, CONFIG1_PROMPTS, arrivals, pack_texts, text, true_len

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LEX_V1 = os.path.join(ROOT, "data", "lexicon_v1.txt")
LEX_MIN = os.path.join(ROOT, "data", "lexicon_min.txt")

#: per-config base of global request ids (requests of different configs never collide)
GID_BASE = {1: 0, 2: 0, 3: 1 << 32, 4: 2 << 32, 5: 3 << 32}
TRACE_STRIDE = 1024  # gid = base + trace * TRACE_STRIDE + i


def load_profiles() -> dict:
    with open(os.path.join(ROOT, "data", "profiles.json")) as f:
        return json.load(f)


def paper_lms() -> list[dict]:
    """The four LMs of the paper's v1 evaluation (DialoGPT, BlenderBot, BART, T5)."""
    return [p for p in load_profiles()["lms"] if p["paper"]]


def regressor(p: dict) -> np.ndarray:
    return np.asarray([float.fromhex(h) for h in p["regressor_hex"]], dtype=np.float32)


def read_lexicon(path: str = LEX_V1) -> bytes:
    with open(path, "rb") as f:
        return f.read()


# ---------------------------------------------------------------- config 1
#: W1 worked fixture: base weights with s = 1, u_max = 40.
W1_REGRESSOR = np.asarray([6, 2, 1.5, 4, 3, 5, 5, 0.5], dtype=np.float32)
#: config-1 ground-truth output lengths (tokens), fixed by this harness
CONFIG1_TRUE_LEN = np.asarray([20, 14, 25, 30, 45, 60, 28, 22], dtype=np.uint16)


def config1_profile() -> dict:
    p = dict(paper_lms()[0])  # DialoGPT
    p.update(u_max=40.0, cores=4)
    return p


def config1():
    data, off = pack_texts(CONFIG1_PROMPTS)
    n = len(CONFIG1_PROMPTS)
    return {"data": data, "offsets": off, "arrival_us": np.zeros(n, np.int64),
            "true_len": CONFIG1_TRUE_LEN.copy(), "trace_off": np.asarray([0, n], np.uint32),
            "profile": config1_profile(), "regressor": W1_REGRESSOR.copy(), "lexicon": read_lexicon(LEX_MIN)}


# ---------------------------------------------------------------- config 2
def config2(n: int = 1 << 20, gid0: int = 0, lm: int = 0):
    """One queue of n requests, all released at 0, one LM (DialoGPT), tight."""
    seed = ROOT_SEED + 2
    data, off, lat = text(seed, GID_BASE[2] + gid0, n, latent=True)
    p = paper_lms()[lm]
    tl = true_len(seed, GID_BASE[2] + gid0, lat, p["scale"], lm)
    return {"data": data, "offsets": off, "arrival_us": np.zeros(n, np.int64), "true_len": tl,
            "seg_off": np.asarray([0, n], np.uint32), "profile": dict(p), "regressor": regressor(p),
            "lexicon": read_lexicon()}


# ---------------------------------------------------------------- traces
def _trace_part(seed, cfg, t, per_trace, f, lm, beta0, step, beta_max):
    g0 = GID_BASE[cfg] + int(t) * TRACE_STRIDE
    d, o, lat = text(seed, g0, per_trace, latent=True)
    return d, o, arrivals(seed, int(t), per_trace, beta0, step, beta_max), true_len(seed, g0, lat, lm["scale"], f)


def traces(cfg: int, trace_ids, per_trace: int, lm_of, beta0=10.0, step=1.0, beta_max=150.0, tightness=1,
           threads: int | None = None):
    """Independent Poisson-ramp traces.  lm_of(trace_id) -> LM index.
    Returns arrays concatenated trace by trace (arrival order within a trace).
    Traces are generated independently (counter-based), on `threads` host
    threads (default: all cores; the result does not depend on it)."""
    from concurrent.futures import ThreadPoolExecutor
    seed = ROOT_SEED + cfg
    lms = paper_lms()
    ids = [int(t) for t in trace_ids]
    lm_idx = [lm_of(t) for t in ids]
    args = [(seed, cfg, t, per_trace, f, lms[f], beta0, step, beta_max) for t, f in zip(ids, lm_idx)]
    nthr = threads or min(32, os.cpu_count() or 1)
    if nthr > 1 and len(ids) > 64:
        with ThreadPoolExecutor(nthr) as ex:  # ctypes calls release the GIL
            parts = list(ex.map(lambda a: _trace_part(*a), args))
    else:
        parts = [_trace_part(*a) for a in args]
    datas, offs, r_all, tl_all = [], [], [], []
    total = 0
    for d, o, r, tl in parts:
        datas.append(d)
        offs.append(o[:-1].astype(np.uint64) + total)
        total += int(o[-1])
        r_all.append(r)
        tl_all.append(tl)
    off = np.concatenate(offs + [np.asarray([total], np.uint64)])
    if total >= 2**32:
        raise OverflowError("trace shard text >= 4 GiB")
    nt = len(lm_idx)
    profiles = []
    for p in lms:
        q = dict(p)
        q["tightness"] = tightness
        profiles.append(q)
    return {"data": np.concatenate(datas) if datas else np.zeros(0, np.uint8), "offsets": off.astype(np.uint32),
            "arrival_us": np.concatenate(r_all) if r_all else np.zeros(0, np.int64),
            "true_len": np.concatenate(tl_all) if tl_all else np.zeros(0, np.uint16),
            "trace_off": (np.arange(nt + 1, dtype=np.uint64) * per_trace).astype(np.uint32),
            "trace_prof": np.asarray(lm_idx, np.uint16), "profiles": profiles, "trace_ids": np.asarray(ids, np.int64),
            "regressors": [regressor(p) for p in lms], "lexicon": read_lexicon()}


def config3(n_traces: int = 4096, per_trace: int = 1000, first: int = 0):
    """4096 traces x 1000 requests; 1024 consecutive traces per LM."""
    per_lm = max(1, 4096 // 4)
    return traces(3, range(first, first + n_traces), per_trace, lambda t: (t // per_lm) % 4)


def config4_shard(rank: int, world: int, n_traces: int = 65536, per_trace: int = 1024, grouped: bool = False):
    """2^26 requests = 65536 traces x 1024, contiguous trace ranges per rank
    (LM of trace t = t mod 4).  grouped=True lists the same traces ordered by
    (LM, t), so that each LM's requests are one contiguous range (one scoring
    launch per LM regressor); traces are independent, so the order does not
    change any per-trace result."""
    lo = rank * n_traces // world
    hi = (rank + 1) * n_traces // world
    ids = range(lo, hi)
    if grouped:
        ids = sorted(ids, key=lambda t: (t % 4, t))
    return traces(4, ids, per_trace, lambda t: t % 4)


#: config 5: arrival-rate multipliers x tightness x policies, plus
#: alpha and b steps on UP+C+O.  SURVEY fixes no rate or tightness for the alpha
#: and b steps; they run at multiplier 8 (the knee of the lighter LMs, SURVEY
#: §8(d) "where overload starts") with loose deadlines, where tasks are not
#: overdue on arrival and the numerator (alpha) and window (b) can matter
CONFIG5_AB_MULT = 8.0
CONFIG5_AB_TIGHTNESS = 2
CONFIG5_MULTS = (0.25, 0.5, 1.0, 2.0, 4.0, 8.0, 16.0, 32.0)
CONFIG5_POLICIES = {
    "FIFO": {"policy": "FIFO", "consolidate": 0, "offload": 0},
    "HPF": {"policy": "HPF", "consolidate": 0, "offload": 0},
    "LUF": {"policy": "LUF", "consolidate": 0, "offload": 0},
    "MUF": {"policy": "MUF", "consolidate": 0, "offload": 0},
    "UP": {"policy": "UP", "consolidate": 0, "offload": 0},
    "UP+C": {"policy": "UP", "consolidate": 1, "offload": 0},
    "UP+C+O": {"policy": "UP", "consolidate": 1, "offload": 1},
}


def config5_points() -> list[dict]:
    """The 154 sweep points: {"mult", "name", "overrides"} (8 x 2 x 7 + 21 alpha + 21 b)."""
    pts = []
    for m in CONFIG5_MULTS:
        for tight in (1, 2):
            for name, ov in CONFIG5_POLICIES.items():
                pts.append({"mult": m, "name": f"{name}/t{tight}", "overrides": dict(ov, tightness=tight)})
    for i in range(21):
        pts.append({"mult": CONFIG5_AB_MULT, "name": f"alpha={i / 10:.1f}",
                    "overrides": dict(CONFIG5_POLICIES["UP+C+O"], alpha=i / 10, tightness=CONFIG5_AB_TIGHTNESS)})
    for b10 in range(10, 31):
        pts.append({"mult": CONFIG5_AB_MULT, "name": f"b={b10 / 10:.1f}",
                    "overrides": dict(CONFIG5_POLICIES["UP+C+O"], b10=b10, tightness=CONFIG5_AB_TIGHTNESS)})
    return pts


def config5_base(first: int, per_lm: int = 64, per_trace: int = 1000):
    """The sweep's traces: 4 x per_lm traces (LM blocks contiguous) at multiplier 1."""
    nt = 4 * per_lm
    return traces(5, range(first, first + nt), per_trace, lambda t: ((t - first) // per_lm) % 4)


def config5_arrivals(d: dict, mult: float) -> np.ndarray:
    """Arrivals of the same traces under the ramp scaled by `mult`
    (rate min(10 m + m j, 150 m) per minute; P:1586-1587 scaled)."""
    seed = ROOT_SEED + 5
    per = int(d["trace_off"][1] - d["trace_off"][0]) if len(d["trace_off"]) > 1 else 0
    return np.concatenate([arrivals(seed, int(t), per, 10.0 * mult, 1.0 * mult, 150.0 * mult)
                           for t in d["trace_ids"]])


# ---------------------------------------------------------------- NEXT-3: periodic release
def periodic_arrivals(trace_off, D_us) -> np.ndarray:
    """Periodic release ("the deadline of one task serves as the
    release time for the subsequent one"): within each trace r_0 = 0 and
    r_{i+1} = r_i + D_i, with D the tasks' relative deadlines (µs) as computed
    by the path (tight: mu*|J|, loose: twice that).  Workload
    construction only (a running sum of the given deadlines)."""
    D = np.asarray(D_us, dtype=np.int64)
    toff = np.asarray(trace_off, dtype=np.int64)
    r = np.zeros(len(D), np.int64)
    for t in range(len(toff) - 1):
        lo, hi = int(toff[t]), int(toff[t + 1])
        if hi > lo + 1:
            r[lo + 1:hi] = np.cumsum(D[lo:hi - 1])
    return r


# ---------------------------------------------------------------- NEXT-3: variance subsets
def variance_subsets(u, size: int, seed: int = ROOT_SEED + 51) -> dict:
    """Three task subsets with small / medium / large variance of the
    uncertainty scores u: `size` tasks nearest the median u; `size`
    tasks drawn from the central two thirds of the u order; `size` tasks drawn
    from all.  Returns index arrays into the pool, each in a seeded random order
    (harness selection only: u comes from the caller)."""
    u = np.asarray(u)
    order = np.argsort(u, kind="stable")
    n = len(u)
    rng = np.random.default_rng(seed)
    mid = n // 2
    small = order[max(0, mid - size // 2): max(0, mid - size // 2) + size]
    central = order[n // 6: n - n // 6]
    medium = rng.choice(central, size=min(size, len(central)), replace=False)
    large = rng.choice(n, size=min(size, n), replace=False)
    for name, v in (("small", small), ("medium", medium), ("large", large)):
        if len(v) != size:  # the caller builds traces of exactly `size` tasks
            raise ValueError(f"variance_subsets: pool of {n} cannot give {size} {name}-variance tasks")
    return {k: rng.permutation(v) for k, v in (("small", small), ("medium", medium), ("large", large))}


# ---------------------------------------------------------------- NEXT-3: malicious tasks
#: appended to a malicious request: crafted words that raise its rule scores (an
#: opener, vague and broad words, coordinators, a comma list, a question), like
#: the paper's crafted inputs that "induce LMs to generate substantially lengthier
#: outputs" (Table "dialogue_adversary" P:763-776)
MALICIOUS_SUFFIX = b" Tell me about the history of art, stuff, countries and the world?"
MALICIOUS_INFLATION = 3  # true output length x3


def with_malicious(d: dict, ratio: float, seed: int = ROOT_SEED + 77) -> dict:
    """A copy of a traces() workload where a seeded `ratio` of the requests
    (0 % to 100 % in steps of 10 %) are malicious: crafted suffix
    appended to the text and the true output length inflated x3 (capped at
    65535).  Arrivals, traces and profiles are unchanged."""
    n = len(d["true_len"])
    rng = np.random.default_rng(seed)
    mal = rng.random(n) < ratio
    data, off = d["data"], d["offsets"].astype(np.int64)
    texts = [bytes(data[off[i]:off[i + 1]]) + (MALICIOUS_SUFFIX if mal[i] else b"") for i in range(n)]
    nd, noff = pack_texts(texts)
    tl = d["true_len"].astype(np.int64)
    tl[mal] = np.minimum(tl[mal] * MALICIOUS_INFLATION, 65535)
    out = dict(d)
    out.update(data=nd, offsets=noff, true_len=tl.astype(np.uint16), malicious=mal)
    return out
