"""rtgen — seeded synthetic workload generator shared by the oracle side and the
CUDA side as their common INPUT (it holds none of the method's arithmetic; see
gen.c's header).  Counter-based: request ``gid`` is identical whichever shard
generates it.

Also holds the fixed prompts of config 1 (BASELINE.json configs[0]): Table 1's
six example sentences, "Can you tell me the history of art?"
 and the dialogue_adversary question.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "librtgen.so")
_SRC = os.path.join(_HERE, "gen.c")

ROOT_SEED = 0x52544C4D  # "RTLM" (SURVEY §8(d) Seeds)

#: config 1 prompts, in this order
CONFIG1_PROMPTS = [
    "John saw a boy in the park with a telescope.",
    "Rice flies like sand.",
    "What's the best way to deal with bats?",
    "Tell me about the history of art.",
    "What are the causes and consequences of poverty in developing countries?",
    "How do cats and dogs differ in behavior, diet, and social interaction?",
    "Can you tell me the history of art?",
    "Not really. Let's talk about food. What do you like to eat? I love fish.",
]

#: latent-count weights of the generator's ground-truth length model (SURVEY §8(d)
#: "Proposed base weights"): [S, Y, M, V, O, P, ntok], intercept c.
BASE_W = (2.0, 1.5, 4.0, 3.0, 5.0, 5.0, 0.5)
BASE_C = 6.0


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        lib.rtgen_text.restype = ctypes.c_uint64
        lib.rtgen_text.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, P, ctypes.c_uint64, P, P]
        lib.rtgen_true_len.restype = None
        lib.rtgen_true_len.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, P, ctypes.c_double,
                                       ctypes.c_double, P, ctypes.c_double, ctypes.c_uint32, P]
        lib.rtgen_arrivals.restype = None
        lib.rtgen_arrivals.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, P]
        lib.rtgen_shuffle.restype = None
        lib.rtgen_shuffle.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, P]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def text(seed: int, gid0: int, n: int, latent: bool = False):
    """Generate requests gid0..gid0+n-1.  Returns (bytes u8[total], offsets u32[n+1]
    [, latent i32[n,7]])."""
    lib = _load()
    off = np.zeros(n + 1, dtype=np.uint64)
    total = lib.rtgen_text(seed, gid0, n, None, 0, _p(off), None)
    buf = np.zeros(max(int(total), 1), dtype=np.uint8)
    lat = np.zeros((n, 7), dtype=np.int32) if latent else None
    lib.rtgen_text(seed, gid0, n, _p(buf), int(total), _p(off), _p(lat) if latent else None)
    if total >= 2**32:
        raise OverflowError("request text >= 4 GiB; split the call (u32 offsets)")
    out = (buf[: int(total)], off.astype(np.uint32))
    return out + (lat,) if latent else out


def pack_texts(texts):
    """Pack explicit strings (UTF-8) into (bytes u8, offsets u32)."""
    bs = [t.encode("utf-8") if isinstance(t, str) else bytes(t) for t in texts]
    off = np.zeros(len(bs) + 1, dtype=np.uint32)
    off[1:] = np.cumsum([len(b) for b in bs], dtype=np.uint64)
    buf = np.frombuffer(b"".join(bs), dtype=np.uint8).copy() if bs else np.zeros(0, np.uint8)
    return buf, off


def true_len(seed: int, gid0: int, latent: np.ndarray, scale: float, lm: int,
             c: float = BASE_C, w=BASE_W, sigma_frac: float = 0.25) -> np.ndarray:
    """Ground-truth output lengths (tokens) from the generator's latent counts."""
    lib = _load()
    latent = np.ascontiguousarray(latent, dtype=np.int32)
    n = latent.shape[0]
    out = np.zeros(n, dtype=np.uint16)
    wv = np.asarray(w, dtype=np.float64)
    lib.rtgen_true_len(seed, gid0, n, _p(latent), float(scale), float(c), _p(wv),
                       float(sigma_frac * scale * c), lm, _p(out))
    return out


def arrivals(seed: int, trace_id: int, n: int, beta0: float = 10.0, step: float = 1.0,
             beta_max: float = 150.0) -> np.ndarray:
    """Poisson arrival times (int64 µs) for one trace: minute j has rate
    min(beta0 + step*j, beta_max) per minute."""
    lib = _load()
    out = np.zeros(n, dtype=np.int64)
    lib.rtgen_arrivals(seed, trace_id, n, float(beta0), float(step), float(beta_max), _p(out))
    return out


def shuffle(seed: int, sid: int, n: int) -> np.ndarray:
    lib = _load()
    out = np.zeros(n, dtype=np.uint32)
    lib.rtgen_shuffle(seed, sid, n, _p(out))
    return out


# ---------------------------------------------------------------- MLP weights (NEXT-1)
MLP_DIMS = (6, 100, 200, 200, 100, 1)


def mlp_weights(seed: int):
    """Random-init weights of the lightweight MLP (no trained weights exist here):
    He-uniform per layer, small uniform biases, float32, row-major [out][in].
    Random numbers only; no arithmetic of the method."""
    rng = np.random.default_rng(seed)
    ws, bs = [], []
    for fan_in, fan_out in zip(MLP_DIMS[:-1], MLP_DIMS[1:]):
        lim = np.sqrt(6.0 / fan_in)
        ws.append(rng.uniform(-lim, lim, (fan_out, fan_in)).astype(np.float32))
        bs.append(rng.uniform(-0.1, 0.1, fan_out).astype(np.float32))
    return ws, bs
