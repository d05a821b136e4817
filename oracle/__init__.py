"""Python wrapper of the RT-LM CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.  The product package
(paper_2309_06619_b200) never imports it and shares no code with it.

The oracle itself is plain C++17 in rtlm_oracle.cpp (steps O1..O8 of
DESIGN.md §3); this file only marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rtlm_oracle.cpp")
_SO = os.path.join(_HERE, "liboracle.so")

POLICY = {"FIFO": 0, "EDF": 1, "HPF": 1, "LUF": 2, "MUF": 3, "SLACK": 4, "UP": 5}


class Profile(ctypes.Structure):
    """The oracle's own profile record (independent of include/rtlm.h)."""
    _fields_ = [
        ("eta_us", ctypes.c_int64), ("mu_us", ctypes.c_int64), ("base_us", ctypes.c_int64),
        ("setup_us", ctypes.c_int64), ("xi_us", ctypes.c_int64),
        ("lambda_", ctypes.c_float), ("alpha", ctypes.c_float), ("tau", ctypes.c_float), ("u_max", ctypes.c_float),
        ("C", ctypes.c_int32), ("b10", ctypes.c_int32), ("tightness", ctypes.c_int32), ("gamma", ctypes.c_int32),
        ("cores", ctypes.c_int32), ("policy", ctypes.c_int32), ("consolidate", ctypes.c_int32),
        ("offload", ctypes.c_int32), ("raw_numerator", ctypes.c_int32), ("pad", ctypes.c_int32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [("sum_resp_us", ctypes.c_int64), ("n", ctypes.c_uint32), ("misses", ctypes.c_uint32)]


def make_profile(d: dict) -> Profile:
    """Build the oracle's profile struct from a plain dict (see data/profiles.json)."""
    p = Profile()
    for k in ("eta_us", "mu_us", "base_us", "setup_us", "xi_us", "C", "b10", "tightness", "gamma", "cores",
              "consolidate", "offload", "raw_numerator"):
        setattr(p, k, int(d[k]))
    p.lambda_ = float(d["lambda"])
    p.alpha = float(d["alpha"])
    p.tau = float(d["tau"])
    p.u_max = float(d["u_max"])
    pol = d["policy"]
    p.policy = POLICY[pol] if isinstance(pol, str) else int(pol)
    return p


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", _SO, _SRC])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        L.orc_lex_load.restype = P
        L.orc_lex_load.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64]
        L.orc_lex_free.argtypes = [P]
        L.orc_lex_size.restype = ctypes.c_uint32
        L.orc_lex_size.argtypes = [P]
        L.orc_lex_lookup.restype = ctypes.c_int
        L.orc_lex_lookup.argtypes = [P, ctypes.c_char_p] + [ctypes.POINTER(ctypes.c_uint32)] * 4
        L.orc_lemma.restype = ctypes.c_int
        L.orc_lemma.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64]
        L.orc_tokenize.restype = ctypes.c_int
        L.orc_tokenize.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64,
                                   ctypes.POINTER(ctypes.c_uint32)]
        L.orc_rule_gen.argtypes = [P, P, P, ctypes.c_uint32, P]
        L.orc_predict.argtypes = [P, ctypes.c_uint32, P, P]
        L.orc_key.argtypes = [P, P, P, P, ctypes.c_uint32, ctypes.POINTER(Profile), P, P]
        L.orc_order.argtypes = [P, P, ctypes.c_uint32, P]
        L.orc_schedule.restype = ctypes.c_uint32
        L.orc_schedule.argtypes = [P, P, P, ctypes.c_uint32, ctypes.POINTER(Profile), ctypes.c_uint32,
                                   P, P, P, P, P]
        L.orc_simulate.argtypes = [P, P, P, P, P, P, ctypes.c_uint32, P, P, P, P]
        L.orc_simulate_util.argtypes = [P, P, P, P, P, P, ctypes.c_uint32, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Lexicon:
    def __init__(self, text: str | bytes):
        L = _load()
        b = text.encode("utf-8") if isinstance(text, str) else text
        err = ctypes.create_string_buffer(512)
        h = L.orc_lex_load(b, len(b), err, 512)
        if not h:
            raise ValueError("lexicon: " + err.value.decode())
        self._h = h

    @classmethod
    def from_file(cls, path: str) -> "Lexicon":
        with open(path, "rb") as f:
            return cls(f.read())

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_lex_free(self._h)
            self._h = None

    def __len__(self):
        return int(_load().orc_lex_size(self._h))

    def lookup(self, word: str):
        """Returns None or dict(flags=..., id=..., senses=..., npos=...) for a surface word."""
        f, i, s, n = (ctypes.c_uint32() for _ in range(4))
        if not _load().orc_lex_lookup(self._h, word.encode(), ctypes.byref(f), ctypes.byref(i), ctypes.byref(s),
                                      ctypes.byref(n)):
            return None
        names = ["vague", "prep", "coord", "noun", "opener", "what", "cause", "broad"]
        return {"flags": {nm for b, nm in enumerate(names) if f.value >> b & 1}, "id": i.value,
                "senses": s.value, "npos": n.value}


def lemma(surface: str) -> str:
    buf = ctypes.create_string_buffer(len(surface) + 8)
    _load().orc_lemma(surface.encode(), buf, len(buf))
    return buf.value.decode()


def tokenize(text: str | bytes):
    """Returns (list of (kind, surface), ndropped); kind 'W' or 'P'."""
    b = text.encode("utf-8") if isinstance(text, str) else text
    buf = ctypes.create_string_buffer(2 * len(b) + 16)
    nd = ctypes.c_uint32()
    cnt = _load().orc_tokenize(b, len(b), buf, len(buf), ctypes.byref(nd))
    if cnt == 0:
        return [], nd.value
    items = buf.raw[: buf.raw.index(b"\0")].split(b"\n")
    return [(it[:1].decode(), it[1:].decode("latin-1")) for it in items], nd.value


def rule_gen(lex: Lexicon, data: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """O1+O2: feat u16[n, 8] = {S, Y, M, V, O, P, ntok, ndropped}."""
    data = np.ascontiguousarray(data, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint32)
    n = len(offsets) - 1
    feat = np.zeros((n, 8), dtype=np.uint16)
    if n:
        _load().orc_rule_gen(lex._h, _p(data if len(data) else np.zeros(1, np.uint8)), _p(offsets), n, _p(feat))
    return feat


def predict(feat: np.ndarray, reg) -> np.ndarray:
    """O3: reg = (c, w0..w6) as float32."""
    feat = np.ascontiguousarray(feat, dtype=np.uint16)
    r = np.ascontiguousarray(np.asarray(reg, dtype=np.float32).reshape(8))
    u = np.zeros(feat.shape[0], dtype=np.float32)
    if len(u):
        _load().orc_predict(_p(feat), feat.shape[0], _p(r), _p(u))
    return u


def key(u, feat, prof: dict, r_us=None, D_in=None):
    """O4: returns (key u64[n], D_us u32[n])."""
    u = np.ascontiguousarray(u, dtype=np.float32)
    n = len(u)
    feat = np.ascontiguousarray(feat if feat is not None else np.zeros((n, 8), np.uint16), dtype=np.uint16)
    r = None if r_us is None else np.ascontiguousarray(r_us, dtype=np.int64)
    Di = None if D_in is None else np.ascontiguousarray(D_in, dtype=np.uint32)
    k = np.zeros(n, dtype=np.uint64)
    D = np.zeros(n, dtype=np.uint32)
    if n:
        p = make_profile(prof)
        _load().orc_key(_p(u), _p(feat), _p(r), _p(Di), n, ctypes.byref(p), _p(k), _p(D))
    return k, D


def order(key_, seg_off) -> np.ndarray:
    key_ = np.ascontiguousarray(key_, dtype=np.uint64)
    seg = np.ascontiguousarray(seg_off, dtype=np.uint32)
    perm = np.zeros(len(key_), dtype=np.uint32)
    _load().orc_order(_p(key_), _p(seg), len(seg) - 1, _p(perm))
    return perm


def schedule(key_, u, seg_off, prof: dict, cores: int | None = None):
    """O5+O6: returns dict(perm, batch_of, slot_of, core_of, seg_batch_off, nbatches)."""
    key_ = np.ascontiguousarray(key_, dtype=np.uint64)
    u = np.ascontiguousarray(u, dtype=np.float32)
    seg = np.ascontiguousarray(seg_off, dtype=np.uint32)
    n = len(key_)
    perm = np.zeros(n, np.uint32)
    batch_of = np.zeros(n, np.uint32)
    slot_of = np.zeros(n, np.uint8)
    core_of = np.zeros(n, np.uint8)
    sbo = np.zeros(len(seg), np.uint32)
    p = make_profile(prof)
    nb = _load().orc_schedule(_p(key_), _p(u), _p(seg), len(seg) - 1, ctypes.byref(p),
                              int(prof["cores"] if cores is None else cores), _p(perm), _p(batch_of), _p(slot_of),
                              _p(core_of), _p(sbo))
    return {"perm": perm, "batch_of": batch_of, "slot_of": slot_of, "core_of": core_of,
            "seg_batch_off": sbo, "nbatches": int(nb)}


UTIL_DTYPE = [("gpu_busy_us", "<i8"), ("cpu_busy_us", "<i8"), ("gpu_batches", "<u4"), ("cpu_tasks", "<u4")]


def simulate(r_us, true_len, u, key_, D_us, trace_off, profiles, trace_prof=None, want_end=False, want_util=False):
    """O7: returns (stats structured array [sum_resp_us, n, misses], end_us or None),
    plus, iff want_util, the per-trace executor busy times accumulated by the
    event loop (UTIL_DTYPE; NEXT-4)."""
    r = np.ascontiguousarray(r_us, dtype=np.int64)
    ln = np.ascontiguousarray(true_len, dtype=np.uint16)
    u = np.ascontiguousarray(u, dtype=np.float32)
    k = np.ascontiguousarray(key_, dtype=np.uint64)
    D = np.ascontiguousarray(D_us, dtype=np.uint32)
    to = np.ascontiguousarray(trace_off, dtype=np.uint32)
    nt = len(to) - 1
    if isinstance(profiles, dict):
        profiles = [profiles]
    parr = (Profile * len(profiles))(*[make_profile(d) for d in profiles])
    tp = None if trace_prof is None else np.ascontiguousarray(trace_prof, dtype=np.uint16)
    st = np.zeros(nt, dtype=[("sum_resp_us", "<i8"), ("n", "<u4"), ("misses", "<u4")])
    end = np.zeros(len(r), dtype=np.int64) if want_end else None
    ut = np.zeros(nt, dtype=UTIL_DTYPE) if want_util else None
    _load().orc_simulate_util(_p(r), _p(ln), _p(u), _p(k), _p(D), _p(to), nt, ctypes.cast(parr, ctypes.c_void_p),
                              _p(tp), _p(st), _p(end), _p(ut))
    return (st, end, ut) if want_util else (st, end)
