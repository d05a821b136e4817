"""paper_2309_06619_b200 — B200-native RT-LM hot path (arXiv 2309.06619).

Thin ctypes binding of include/rtlm.h.  Every function only marshals torch
CUDA tensors into device pointers plus the current CUDA stream; every step of
the path runs in the CUDA kernels of librtlm.so.  There is no CPU fallback:
if the library cannot be loaded or no GPU is present, calls raise.

Call names follow the boundary: score (RuleGen, Eq. 1), predict (m_theta),
key (Eq. 2/3 priority + offload class), score_key (fused), schedule
(Alg. 1 online part), simulate (trace replay), reduce_stats (aggregation).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RTLM_LIB", os.path.join(_HERE, "librtlm.so"))  # RTLM_LIB: an alternative build (experiments)
CSRC = os.path.join(_HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(_HERE), "include")

POLICY = {"FIFO": 0, "EDF": 1, "HPF": 1, "LUF": 2, "MUF": 3, "SLACK": 4, "UP": 5}
RT_STATUS = {0: "RT_OK", 1: "RT_EINVAL", 2: "RT_ELEXICON", 3: "RT_ENOMEM", 4: "RT_ECUDA", 5: "RT_EOVERFLOW"}
EXPORTS = ["rt_create", "rt_destroy", "rt_last_error", "rt_get_flags", "rt_abi_version", "rt_lexicon_size",
           "rt_score", "rt_predict", "rt_key", "rt_score_key", "rt_schedule", "rt_simulate", "rt_reduce_stats", "rt_launch_count",
           "rt_set_mlp", "rt_predict_mlp", "rt_set_mlp_precision", "rt_fit_rule", "rt_quantile", "rt_trace_report",
           "rt_trace_utilization", "rt_set_sm_limit", "rt_score_schedule_host",
           "rt_schedule_deadlines", "rt_train_mlp", "rt_get_mlp"]
NO_BATCH = 0xFFFFFFFF


class RtlmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{RT_STATUS.get(status, status)}: {msg}")
        self.status = status


class Regressor(ctypes.Structure):
    _fields_ = [("c", ctypes.c_float), ("w", ctypes.c_float * 7)]


class Profile(ctypes.Structure):
    _fields_ = [
        ("eta_us", ctypes.c_int64), ("mu_us", ctypes.c_int64), ("base_us", ctypes.c_int64),
        ("setup_us", ctypes.c_int64), ("xi_us", ctypes.c_int64),
        ("lambda_", ctypes.c_float), ("alpha", ctypes.c_float), ("tau", ctypes.c_float), ("u_max", ctypes.c_float),
        ("C", ctypes.c_int32), ("b10", ctypes.c_int32), ("tightness", ctypes.c_int32), ("gamma", ctypes.c_int32),
        ("cores", ctypes.c_int32), ("policy", ctypes.c_int32), ("consolidate", ctypes.c_int32),
        ("offload", ctypes.c_int32), ("raw_numerator", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


def make_profile(d: dict) -> Profile:
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
    p.reserved = 0
    return p


class Mlp(ctypes.Structure):
    """rt_mlp: host fp32 weights [out][in] and biases of the 6-100-200-200-100-1 MLP."""
    _fields_ = [("w", ctypes.c_void_p * 5), ("b", ctypes.c_void_p * 5)]


MLP_DIMS = (6, 100, 200, 200, 100, 1)


def make_regressor(coefs) -> Regressor:
    c = np.asarray(coefs, dtype=np.float32).reshape(8)
    r = Regressor()
    r.c = float(c[0])
    for k in range(7):
        r.w[k] = float(c[1 + k])
    return r


_lib = None


def load_library(path: str = LIB_PATH):
    """Loads librtlm.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RtlmError(4, f"{path} not built (run __graft_entry__.build())")
    L = ctypes.CDLL(path)
    V, P, U32, I32, SZ = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int, ctypes.c_size_t
    L.rt_create.restype = I32
    L.rt_create.argtypes = [I32, ctypes.c_char_p, SZ, ctypes.POINTER(V)]
    L.rt_destroy.restype = I32
    L.rt_destroy.argtypes = [V]
    L.rt_last_error.restype = ctypes.c_char_p
    L.rt_last_error.argtypes = [V]
    L.rt_get_flags.restype = I32
    L.rt_get_flags.argtypes = [V, ctypes.POINTER(U32)]
    L.rt_abi_version.restype = I32
    L.rt_launch_count.restype = ctypes.c_uint64
    L.rt_lexicon_size.restype = U32
    L.rt_lexicon_size.argtypes = [V]
    L.rt_set_sm_limit.restype = I32
    L.rt_set_sm_limit.argtypes = [V, U32]
    L.rt_score.restype = I32
    L.rt_score.argtypes = [V, P, P, U32, P, V]
    L.rt_predict.restype = I32
    L.rt_predict.argtypes = [V, P, U32, ctypes.POINTER(Regressor), P, V]
    L.rt_key.restype = I32
    L.rt_key.argtypes = [V, P, P, P, P, U32, ctypes.POINTER(Profile), P, P, V]
    L.rt_score_key.restype = I32
    L.rt_score_key.argtypes = [V, P, P, U32, ctypes.POINTER(Regressor), ctypes.POINTER(Profile), P, P, P, P, P, P, V]
    L.rt_schedule.restype = I32
    L.rt_schedule.argtypes = [V, P, P, P, U32, ctypes.POINTER(Profile), U32, P, P, P, P, P, V]
    L.rt_simulate.restype = I32
    L.rt_simulate.argtypes = [V, P, P, P, P, P, P, U32, P, U32, P, P, P, V]
    L.rt_reduce_stats.restype = I32
    L.rt_reduce_stats.argtypes = [V, P, U32, P, U32, P, V]
    L.rt_set_mlp.restype = I32
    L.rt_set_mlp.argtypes = [V, ctypes.POINTER(Mlp)]
    L.rt_predict_mlp.restype = I32
    L.rt_predict_mlp.argtypes = [V, P, U32, P, V]
    L.rt_train_mlp.restype = I32
    L.rt_train_mlp.argtypes = [V, P, P, U32, U32, U32, ctypes.c_float, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double), V]
    L.rt_get_mlp.restype = I32
    L.rt_get_mlp.argtypes = [V, ctypes.POINTER(P * 5), ctypes.POINTER(P * 5)]
    L.rt_set_mlp_precision.restype = I32
    L.rt_set_mlp_precision.argtypes = [V, ctypes.c_int]
    L.rt_fit_rule.restype = I32
    L.rt_fit_rule.argtypes = [V, P, P, U32, P, V]
    L.rt_quantile.restype = I32
    L.rt_quantile.argtypes = [V, P, U32, ctypes.c_double, P, V]
    L.rt_trace_report.restype = I32
    L.rt_trace_report.argtypes = [V, P, P, P, U32, P, V]
    L.rt_trace_utilization.restype = I32
    L.rt_trace_utilization.argtypes = [V, P, P, P, P, U32, P, U32, P, P, V]
    L.rt_schedule_deadlines.restype = I32
    L.rt_schedule_deadlines.argtypes = [V, P, P, P, P, U32, ctypes.POINTER(Profile), U32, P, P, P, P, P, V]
    L.rt_score_schedule_host.restype = I32
    L.rt_score_schedule_host.argtypes = [V, P, P, U32, ctypes.POINTER(Regressor), ctypes.POINTER(Profile), U32,
                                         P, P, P, V]
    _lib = L
    return L


def launch_count() -> int:
    """Kernel launches issued by librtlm.so so far (this process)."""
    return int(load_library().rt_launch_count())


def _torch():
    import torch
    return torch


def _ptr(t, dtype=None, name="tensor"):
    """Device pointer of a contiguous CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must have dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _hptr(t, dtype, name="tensor"):
    """Host pointer of a contiguous CPU tensor (page-locked for asynchronous copies)."""
    torch = _torch()
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise TypeError(f"{name} must be a CPU tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must have dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


class Context:
    """One rt_ctx (one device, one lexicon)."""

    def __init__(self, lexicon: bytes | str, device: int = 0):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RtlmError(4, "no CUDA device: the RT-LM hot path has no CPU fallback")
        self._L = load_library()
        self.device = torch.device("cuda", device)
        b = lexicon.encode("utf-8") if isinstance(lexicon, str) else bytes(lexicon)
        h = ctypes.c_void_p()
        st = self._L.rt_create(device, b, len(b), ctypes.byref(h))
        self._h = h
        if st != 0:
            msg = self._L.rt_last_error(h).decode() if h else "rt_create failed"
            self.close()
            raise RtlmError(st, msg)

    def close(self):
        if getattr(self, "_h", None):
            self._L.rt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ helpers
    def _stream(self):
        torch = _torch()
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _check(self, st):
        if st != 0:
            raise RtlmError(st, self._L.rt_last_error(self._h).decode())

    def _empty(self, shape, dtype):
        return _torch().empty(shape, dtype=dtype, device=self.device)

    @property
    def lexicon_size(self) -> int:
        return int(self._L.rt_lexicon_size(self._h))

    def set_sm_limit(self, max_ctas: int) -> None:
        """Caps the CTAs of this context's persistent kernels (rt_set_sm_limit; 0 = one per SM)."""
        self._check(self._L.rt_set_sm_limit(self._h, int(max_ctas)))

    def flags(self) -> int:
        f = ctypes.c_uint32()
        self._check(self._L.rt_get_flags(self._h, ctypes.byref(f)))
        return f.value

    # ------------------------------------------------------------ calls
    def score(self, data, offsets, feat=None):
        """rt_score: uint8 bytes + int32-viewed uint32 offsets -> feat uint16-as-int16 [n, 8]."""
        torch = _torch()
        n = offsets.numel() - 1
        if feat is None:
            feat = self._empty((max(n, 0), 8), torch.int16)
        self._check(self._L.rt_score(self._h, _ptr(data, torch.uint8, "data"), _ptr(offsets, torch.int32, "offsets"),
                                     n, _ptr(feat, torch.int16, "feat"), self._stream()))
        return feat

    def predict(self, feat, reg, u=None):
        torch = _torch()
        n = feat.shape[0]
        if u is None:
            u = self._empty((n,), torch.float32)
        r = make_regressor(reg)
        self._check(self._L.rt_predict(self._h, _ptr(feat, torch.int16, "feat"), n, ctypes.byref(r),
                                       _ptr(u, torch.float32, "u"), self._stream()))
        return u

    def set_mlp(self, weights, biases):
        """rt_set_mlp: weights[l] fp32 [out][in], biases[l] fp32 [out] (copied at call time)."""
        ws = [np.ascontiguousarray(w, dtype=np.float32) for w in weights]
        bs = [np.ascontiguousarray(b, dtype=np.float32) for b in biases]
        for l, (w, b) in enumerate(zip(ws, bs)):
            if w.shape != (MLP_DIMS[l + 1], MLP_DIMS[l]) or b.shape != (MLP_DIMS[l + 1],):
                raise ValueError(f"layer {l}: expected {(MLP_DIMS[l + 1], MLP_DIMS[l])} / {(MLP_DIMS[l + 1],)}")
        m = Mlp()
        for l in range(5):
            m.w[l] = ws[l].ctypes.data
            m.b[l] = bs[l].ctypes.data
        self._check(self._L.rt_set_mlp(self._h, ctypes.byref(m)))

    def train_mlp(self, feat, y, epochs: int, batch: int, lr: float, seed: int = 0):
        """rt_train_mlp (NEXT-2): Adam on the MSE of the context's MLP (from the weights
        of set_mlp) over feat uint16-as-int16 [n, 8] and y float32 [n]; returns the
        per-epoch losses (numpy float64).  Synchronizes the current stream."""
        torch = _torch()
        n = feat.shape[0]
        losses = np.zeros(max(int(epochs), 1), np.float64)
        self._check(self._L.rt_train_mlp(self._h, _ptr(feat, torch.int16, "feat"), _ptr(y, torch.float32, "y"), n,
                                         int(epochs), int(batch), float(lr), int(seed),
                                         losses.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), self._stream()))
        return losses[:int(epochs)]

    def get_mlp(self):
        """rt_get_mlp: the context's current MLP weights -> (weights, biases), fp32 numpy."""
        ws = [np.zeros((MLP_DIMS[l + 1], MLP_DIMS[l]), np.float32) for l in range(5)]
        bs = [np.zeros(MLP_DIMS[l + 1], np.float32) for l in range(5)]
        pw = (ctypes.c_void_p * 5)(*[w.ctypes.data for w in ws])
        pb = (ctypes.c_void_p * 5)(*[b.ctypes.data for b in bs])
        self._check(self._L.rt_get_mlp(self._h, ctypes.byref(pw), ctypes.byref(pb)))
        return ws, bs

    def set_mlp_precision(self, precision: str) -> None:
        """rt_set_mlp_precision: "fp32" (default, CUDA-core binary32), "tf32x3"
        (tcgen05 3xTF32, fp32-accurate) or "bf16" (tcgen05, opt-in fast mode)."""
        self._check(self._L.rt_set_mlp_precision(self._h, {"fp32": 0, "bf16": 1, "tf32x3": 2}[precision]))

    def predict_mlp(self, feat, u=None):
        """rt_predict_mlp: feat uint16-as-int16 [n, 8] -> u float32 [n]."""
        torch = _torch()
        n = feat.shape[0]
        if u is None:
            u = self._empty((n,), torch.float32)
        self._check(self._L.rt_predict_mlp(self._h, _ptr(feat, torch.int16, "feat"), n, _ptr(u, torch.float32, "u"),
                                           self._stream()))
        return u

    def fit_rule(self, feat, target, out=None):
        """rt_fit_rule: feat uint16-as-int16 [n, 8], target float32 [n] -> float64 [8]
        = (c, w_S, w_Y, w_M, w_V, w_O, w_P, cond)."""
        torch = _torch()
        if out is None:
            out = self._empty((8,), torch.float64)
        self._check(self._L.rt_fit_rule(self._h, _ptr(feat, torch.int16, "feat"), _ptr(target, torch.float32, "target"),
                                        feat.shape[0], _ptr(out, torch.float64, "out"), self._stream()))
        return out

    def quantile(self, u, k: float, out=None):
        """rt_quantile: -> float32 [2] = (nearest-rank k-quantile, max)."""
        torch = _torch()
        if out is None:
            out = self._empty((2,), torch.float32)
        self._check(self._L.rt_quantile(self._h, _ptr(u, torch.float32, "u"), u.numel(), float(k),
                                        _ptr(out, torch.float32, "out"), self._stream()))
        return out

    def trace_report(self, arrival, end_us, trace_off, out=None):
        """rt_trace_report: -> int64 [nt, 4] = (max_resp_us, p95_resp_us, makespan_us, n | reserved << 32)."""
        torch = _torch()
        toff = np.ascontiguousarray(trace_off, dtype=np.uint32)
        nt = len(toff) - 1
        if out is None:
            out = self._empty((nt, 4), torch.int64)
        self._check(self._L.rt_trace_report(self._h, _ptr(arrival, torch.int64, "arrival"),
                                            _ptr(end_us, torch.int64, "end_us"),
                                            toff.ctypes.data_as(ctypes.c_void_p), nt, _ptr(out, torch.int64, "out"),
                                            self._stream()))
        return out

    def trace_utilization(self, true_len, key, end_us, trace_off, profiles, trace_prof=None, out=None):
        """rt_trace_utilization: -> int64 [nt, 3] = (gpu_busy_us, cpu_busy_us, gpu_batches | cpu_tasks << 32)."""
        torch = _torch()
        toff = np.ascontiguousarray(trace_off, dtype=np.uint32)
        nt = len(toff) - 1
        if isinstance(profiles, dict):
            profiles = [profiles]
        parr = (Profile * len(profiles))(*[make_profile(d) for d in profiles])
        if out is None:
            out = self._empty((nt, 3), torch.int64)
        self._check(self._L.rt_trace_utilization(self._h, _ptr(true_len, torch.int16, "true_len"),
                                                 _ptr(key, torch.int64, "key"), _ptr(end_us, torch.int64, "end_us"),
                                                 toff.ctypes.data_as(ctypes.c_void_p), nt,
                                                 ctypes.cast(parr, ctypes.c_void_p), len(profiles),
                                                 _ptr(trace_prof, torch.int16, "trace_prof"),
                                                 _ptr(out, torch.int64, "out"), self._stream()))
        return out

    def key(self, u, prof: dict, feat=None, arrival=None, D_in=None, key=None, D_out=None):
        torch = _torch()
        n = u.numel()
        key = self._empty((n,), torch.int64) if key is None else key
        D_out = self._empty((n,), torch.int32) if D_out is None else D_out
        p = make_profile(prof)
        self._check(self._L.rt_key(self._h, _ptr(u, torch.float32, "u"), _ptr(feat, torch.int16, "feat"),
                                   _ptr(arrival, torch.int64, "arrival"), _ptr(D_in, torch.int32, "D_in"), n,
                                   ctypes.byref(p), _ptr(key, torch.int64, "key"), _ptr(D_out, torch.int32, "D_out"),
                                   self._stream()))
        return key, D_out

    def score_key(self, data, offsets, reg, prof: dict, arrival=None, D_in=None, want_feat=False, want_D=True,
                  out=None):
        """Fused rt_score_key.  Returns dict(u, key[, D][, feat]).  `out` may pass preallocated tensors."""
        torch = _torch()
        n = offsets.numel() - 1
        out = dict(out or {})
        u = out.get("u") if out.get("u") is not None else self._empty((n,), torch.float32)
        key = out.get("key") if out.get("key") is not None else self._empty((n,), torch.int64)
        D = out.get("D") if want_D else None
        if want_D and D is None:
            D = self._empty((n,), torch.int32)
        feat = out.get("feat") if want_feat else None
        if want_feat and feat is None:
            feat = self._empty((n, 8), torch.int16)
        r = make_regressor(reg)
        p = make_profile(prof)
        self._check(self._L.rt_score_key(self._h, _ptr(data, torch.uint8, "data"),
                                         _ptr(offsets, torch.int32, "offsets"), n, ctypes.byref(r), ctypes.byref(p),
                                         _ptr(arrival, torch.int64, "arrival"), _ptr(D_in, torch.int32, "D_in"),
                                         _ptr(feat, torch.int16, "feat"), _ptr(u, torch.float32, "u"),
                                         _ptr(key, torch.int64, "key"), _ptr(D, torch.int32, "D"), self._stream()))
        res = {"u": u, "key": key}
        if want_D:
            res["D"] = D
        if want_feat:
            res["feat"] = feat
        return res

    def score_schedule_host(self, h_bytes, h_offsets, reg, prof: dict, out, cores: int | None = None):
        """rt_score_schedule_host: one queue end to end from HOST tensors (pinned
        for asynchronous copies): h_bytes u8, h_offsets int32 (u32 bits, n+1);
        `out` = dict of host tensors batch_of (int32), slot_of (uint8), core_of
        (uint8), valid after the current stream synchronises."""
        torch = _torch()
        n = h_offsets.numel() - 1
        r = make_regressor(reg)
        p = make_profile(prof)
        c = int(prof["cores"] if cores is None else cores)
        self._check(self._L.rt_score_schedule_host(
            self._h, _hptr(h_bytes, torch.uint8, "h_bytes"), _hptr(h_offsets, torch.int32, "h_offsets"), n,
            ctypes.byref(r), ctypes.byref(p), c, _hptr(out["batch_of"], torch.int32, "batch_of"),
            _hptr(out["slot_of"], torch.uint8, "slot_of"), _hptr(out["core_of"], torch.uint8, "core_of"),
            self._stream()))
        return out

    def schedule_deadlines(self, u, D, seg_off, prof: dict, arrival=None, cores: int | None = None):
        """rt_schedule_deadlines: keys from u and relative deadlines D (int32 view of
        u32 µs) in-call, then the one-pass schedule.  Returns dict of device tensors."""
        torch = _torch()
        so = np.ascontiguousarray(np.asarray(seg_off, dtype=np.uint32))
        nq = len(so) - 1
        n = int(so[-1])
        out = {"perm": self._empty((n,), torch.int32), "batch_of": self._empty((n,), torch.int32),
               "slot_of": self._empty((n,), torch.uint8), "core_of": self._empty((n,), torch.uint8),
               "seg_batch_off": self._empty((nq + 1,), torch.int32)}
        p = make_profile(prof)
        c = int(prof["cores"] if cores is None else cores)
        self._check(self._L.rt_schedule_deadlines(
            self._h, _ptr(u, torch.float32, "u"), _ptr(D, torch.int32, "D"), _ptr(arrival, torch.int64, "arrival"),
            so.ctypes.data_as(ctypes.c_void_p), nq, ctypes.byref(p), c, _ptr(out["perm"], torch.int32, "perm"),
            _ptr(out["batch_of"], torch.int32, "batch_of"), _ptr(out["slot_of"], torch.uint8, "slot_of"),
            _ptr(out["core_of"], torch.uint8, "core_of"), _ptr(out["seg_batch_off"], torch.int32, "seg_batch_off"),
            self._stream()))
        return out

    def schedule(self, key, u, seg_off, prof: dict, cores: int | None = None, out=None):
        """rt_schedule.  seg_off: host array (nq+1).  Returns dict of device tensors."""
        torch = _torch()
        so = np.ascontiguousarray(np.asarray(seg_off, dtype=np.uint32))
        nq = len(so) - 1
        n = int(so[-1])
        out = dict(out or {})
        perm = out.get("perm") if out.get("perm") is not None else self._empty((n,), torch.int32)
        batch_of = out.get("batch_of") if out.get("batch_of") is not None else self._empty((n,), torch.int32)
        slot_of = out.get("slot_of") if out.get("slot_of") is not None else self._empty((n,), torch.uint8)
        core_of = out.get("core_of") if out.get("core_of") is not None else self._empty((n,), torch.uint8)
        sbo = out.get("seg_batch_off") if out.get("seg_batch_off") is not None else self._empty((nq + 1,), torch.int32)
        p = make_profile(prof)
        c = int(prof["cores"] if cores is None else cores)
        self._check(self._L.rt_schedule(self._h, _ptr(key, torch.int64, "key"), _ptr(u, torch.float32, "u"),
                                        so.ctypes.data_as(ctypes.c_void_p), nq, ctypes.byref(p), c,
                                        _ptr(perm, torch.int32, "perm"), _ptr(batch_of, torch.int32, "batch_of"),
                                        _ptr(slot_of, torch.uint8, "slot_of"), _ptr(core_of, torch.uint8, "core_of"),
                                        _ptr(sbo, torch.int32, "seg_batch_off"), self._stream()))
        return {"perm": perm, "batch_of": batch_of, "slot_of": slot_of, "core_of": core_of, "seg_batch_off": sbo}

    def simulate(self, arrival, true_len, u, key, D, trace_off, profiles, trace_prof=None, want_end=False,
                 stats=None):
        """rt_simulate.  trace_off: host array (nt+1); profiles: list of dicts.
        Returns (stats int64 [nt, 2] raw rt_trace_stats, end_us or None)."""
        torch = _torch()
        to = np.ascontiguousarray(np.asarray(trace_off, dtype=np.uint32))
        nt = len(to) - 1
        if isinstance(profiles, dict):
            profiles = [profiles]
        parr = (Profile * len(profiles))(*[make_profile(d) for d in profiles])
        stats = self._empty((nt, 2), torch.int64) if stats is None else stats
        end = self._empty((int(to[-1]),), torch.int64) if want_end else None
        self._check(self._L.rt_simulate(self._h, _ptr(arrival, torch.int64, "arrival"),
                                        _ptr(true_len, torch.int16, "true_len"), _ptr(u, torch.float32, "u"),
                                        _ptr(key, torch.int64, "key"), _ptr(D, torch.int32, "D"),
                                        to.ctypes.data_as(ctypes.c_void_p), nt,
                                        ctypes.cast(parr, ctypes.c_void_p), len(profiles),
                                        _ptr(trace_prof, torch.int16, "trace_prof"), _ptr(stats, torch.int64, "stats"),
                                        _ptr(end, torch.int64, "end_us"), self._stream()))
        return stats, end

    def reduce_stats(self, stats, group_of=None, ngroups: int = 1, sums=None):
        torch = _torch()
        nt = stats.shape[0]
        if sums is None:
            sums = torch.zeros((ngroups, 3), dtype=torch.int64, device=self.device)
        self._check(self._L.rt_reduce_stats(self._h, _ptr(stats, torch.int64, "stats"), nt,
                                            _ptr(group_of, torch.int16, "group_of"), ngroups,
                                            _ptr(sums, torch.int64, "sums"), self._stream()))
        return sums


def decode_stats(stats) -> np.ndarray:
    """Raw rt_trace_stats rows (int64 [nt, 2]) -> structured numpy array."""
    s = stats.detach().cpu().numpy() if hasattr(stats, "detach") else np.asarray(stats)
    out = np.zeros(s.shape[0], dtype=[("sum_resp_us", "<i8"), ("n", "<u4"), ("misses", "<u4")])
    out["sum_resp_us"] = s[:, 0]
    out["n"] = (s[:, 1].astype(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    out["misses"] = (s[:, 1].astype(np.uint64) >> np.uint64(32)).astype(np.uint32)
    return out
