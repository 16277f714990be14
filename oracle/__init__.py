"""fp64 CPU oracle for LongFlow's fused decode step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package
``paper_2603_11504_b200`` never imports it, and the two share no code: the arithmetic
lives in ``oracle/lfo.c`` (plain sequential fp64 loops, see its header for the
paper citations of every step), this module only marshals numpy arrays through ctypes.

Citation key: P:n = PAPER.md line n (Eq. 1, Eq. 4, Eq. 5 P:132,
Eq. 6, Alg. 1, Fig. 2); readings R1..R17 are listed in DESIGN.md.
All functions are pinned by tests/test_oracle_pins.py (none is "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lfo.c")
_LIB = os.path.join(_HERE, "liblfo.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared", "-pthread"]


def build(force: bool = False) -> str:
    """Compile oracle/lfo.c -> oracle/liblfo.so with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            i, dbl = ctypes.c_int, ctypes.c_double
            lib.lfo_unit_attend.argtypes = [i, i, i, dbl, P, P, P, P, P, P, P, P, P, P]
            lib.lfo_unit_attend.restype = i
            lib.lfo_step_compute.argtypes = [i, i, i, i, i, dbl, P, P, P, P, P, P, P, P, P, i]
            lib.lfo_step_compute.restype = i
            lib.lfo_step_apply.argtypes = [i, i, i, i, P, P, P, P, P, P]
            lib.lfo_step_apply.restype = i
            lib.lfo_step_deferred.argtypes = [i, i, i, i, i, dbl, P, P, P, P, P, P, P, P, P, P, i, i]
            lib.lfo_step_deferred.restype = i
            lib.lfo_snapkv_select.argtypes = [i, i, i, i, i, i, dbl, P, P, P, P, P]
            lib.lfo_snapkv_select.restype = i
            lib.lfo_exact_objective.argtypes = [i, i, i, dbl, P, P, P, P, P, P]
            lib.lfo_exact_objective.restype = i
            _lib = lib
    return _lib


def _u16(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype != np.uint16:
        raise TypeError(f"expected bf16 bit patterns as uint16, got {a.dtype}")
    return a


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    pass


def unit_attend(q, K, V, k_new=None, v_new=None, scale=None):
    """One unit: Eq. 1 attention + Eq. 6 LongFlowScore (mean over the G query heads).

    q: uint16 [G][d]; K, V: uint16 [n][d]; k_new/v_new: uint16 [d] or None (cache only,
    Alg. 1's input form P:507).  Returns dict(out [G][d], alpha [G][n+1], scores [n],
    m [G], Z [G], slot) -- slot = lowest-index argmin, -1 if n == 0.
    """
    lib = _load()
    q = _u16(q)
    G, d = q.shape
    K = _u16(K).reshape(-1, d)
    V = _u16(V).reshape(-1, d)
    n = K.shape[0]
    if (k_new is None) != (v_new is None):
        raise ValueError("k_new and v_new must both be given or both be None")
    kn = None if k_new is None else _u16(k_new).reshape(d)
    vn = None if v_new is None else _u16(v_new).reshape(d)
    sc = (1.0 / np.sqrt(d)) if scale is None else float(scale)
    out = np.zeros((G, d), np.float64)
    alpha = np.zeros((G, n + 1), np.float64)
    scores = np.zeros((max(n, 1),), np.float64)
    m = np.zeros((G,), np.float64)
    Z = np.zeros((G,), np.float64)
    r = lib.lfo_unit_attend(G, d, n, sc, _p(q), _p(K), _p(V), _p(kn), _p(vn),
                            _p(out), _p(alpha), _p(scores), _p(m), _p(Z))
    if r == -2:
        raise OracleError("empty attention support")
    if r < -1:
        raise OracleError(f"oracle error {r}")
    if kn is None:
        alpha = alpha[:, :n]
    return dict(out=out, alpha=alpha, scores=scores[:n], m=m, Z=Z, slot=int(r))


class OracleCache:
    """The oracle's own copy of a static KV cache and its step protocol.

    K, V: uint16 [B][Hkv][N][d]; n_valid: int32 [B][Hkv] (R11: slots fill lowest-first).
    """

    def __init__(self, B, Hq, Hkv, d, N, scale=None, nthreads=1):
        if Hq % Hkv:
            raise ValueError("Hq % Hkv != 0")
        if N < 2 or d < 1:
            raise ValueError("budget < 2 or head_dim < 1")
        self.B, self.Hq, self.Hkv, self.d, self.N = B, Hq, Hkv, d, N
        self.G = Hq // Hkv
        self.scale = (1.0 / np.sqrt(d)) if not scale else float(scale)
        self.K = np.zeros((B, Hkv, N, d), np.uint16)
        self.V = np.zeros((B, Hkv, N, d), np.uint16)
        self.n_valid = np.zeros((B, Hkv), np.int32)
        self.pend = np.full((B, Hkv), -1, np.int32)
        self.nthreads = nthreads

    def prefill(self, b, k, v):
        """Slots [0, n) of every kv head of sequence b <- rows of k, v ([Hkv][n][d])."""
        k = _u16(k)
        v = _u16(v)
        n = k.shape[1]
        if n > self.N:
            raise OracleError("prefill exceeds budget; compress first")
        self.K[b, :, :n] = k
        self.V[b, :, :n] = v
        self.n_valid[b, :] = n
        self.pend[b, :] = -1   # deferred modes: no victim chosen yet for this sequence (R26)

    def compute(self, q, k_new, v_new, want_scores=True):
        """Same-step mode (R1), no mutation.  Returns (out fp64 [B][Hq][d], slot int32 [B][Hkv],
        scores fp64 [B][Hkv][N] or None)."""
        lib = _load()
        B, Hq, Hkv, d, N = self.B, self.Hq, self.Hkv, self.d, self.N
        q, k_new, v_new = _u16(q), _u16(k_new), _u16(v_new)
        out = np.zeros((B, Hq, d), np.float64)
        slot = np.zeros((B, Hkv), np.int32)
        scores = np.zeros((B, Hkv, N), np.float64) if want_scores else None
        r = lib.lfo_step_compute(B, Hq, Hkv, d, N, self.scale, _p(self.K), _p(self.V),
                                 _p(self.n_valid), _p(q), _p(k_new), _p(v_new), _p(out),
                                 _p(slot), _p(scores), self.nthreads)
        if r:
            raise OracleError(f"lfo_step_compute failed: {r}")
        return out, slot, scores

    def apply(self, k_new, v_new, slot):
        lib = _load()
        slot = np.ascontiguousarray(slot, np.int32)
        r = lib.lfo_step_apply(self.B, self.Hkv, self.d, self.N, _p(self.K), _p(self.V),
                               _p(self.n_valid), _p(_u16(k_new)), _p(_u16(v_new)), _p(slot))
        if r:
            raise OracleError(f"lfo_step_apply failed: {r}")

    def step(self, q, k_new, v_new):
        out, slot, scores = self.compute(q, k_new, v_new)
        self.apply(k_new, v_new, slot)
        return out, slot, scores

    def step_deferred(self, q, k_new, v_new, exclude_newest=False):
        """Deferred mode (Fig. 2 literal).  Returns (out, written_slot, next_pend, scores)."""
        lib = _load()
        B, Hq, Hkv, d, N = self.B, self.Hq, self.Hkv, self.d, self.N
        out = np.zeros((B, Hq, d), np.float64)
        written = np.zeros((B, Hkv), np.int32)
        scores = np.zeros((B, Hkv, N), np.float64)
        r = lib.lfo_step_deferred(B, Hq, Hkv, d, N, self.scale, _p(self.K), _p(self.V),
                                  _p(self.n_valid), _p(self.pend), _p(_u16(q)), _p(_u16(k_new)),
                                  _p(_u16(v_new)), _p(out), _p(written), _p(scores),
                                  int(bool(exclude_newest)), self.nthreads)
        if r:
            raise OracleError(f"lfo_step_deferred failed: {r}")
        return out, written, self.pend.copy(), scores


def snapkv_select(q_obs, K, budget, pool_kernel=7, scale=None):
    """SnapKV prefill selection for one unit (NEXT-f3; readings R22-R24).
    q_obs: uint16 [G][w][d] (the last w prompt positions' queries of the group), K: uint16 [n][d].
    Returns dict(kept int32 [budget] ascending, score [n-w], pooled [n-w])."""
    lib = _load()
    q_obs = _u16(q_obs)
    G, w, d = q_obs.shape
    K = _u16(K).reshape(-1, d)
    n = K.shape[0]
    sc = (1.0 / np.sqrt(d)) if scale is None else float(scale)
    kept = np.zeros((budget,), np.int32)
    score = np.zeros((max(n - w, 1),), np.float64)
    pooled = np.zeros((max(n - w, 1),), np.float64)
    r = lib.lfo_snapkv_select(G, d, n, w, pool_kernel, budget, sc, _p(q_obs), _p(K), _p(kept), _p(score), _p(pooled))
    if r < 0:
        raise OracleError(f"lfo_snapkv_select failed: {r}")
    return dict(kept=kept, score=score[:n - w], pooled=pooled[:n - w])


def exact_objective(q, K, V, k_new=None, v_new=None, scale=None):
    """NEXT-f4 by brute force (Eq. 3's right-hand side with the current query): for
    every cached token i, the unit re-attended without it; E_i = mean_g ||o_g - o_g^(\\i)||^2.
    q: uint16 [G][d]; K, V: uint16 [n][d]; k_new/v_new: uint16 [d] or None.  Returns E fp64 [n]."""
    lib = _load()
    q = _u16(q)
    G, d = q.shape
    K = _u16(K).reshape(-1, d)
    V = _u16(V).reshape(-1, d)
    n = K.shape[0]
    kn = None if k_new is None else _u16(k_new).reshape(d)
    vn = None if v_new is None else _u16(v_new).reshape(d)
    sc = (1.0 / np.sqrt(d)) if scale is None else float(scale)
    E = np.zeros((max(n, 1),), np.float64)
    r = lib.lfo_exact_objective(G, d, n, sc, _p(q), _p(K), _p(V), _p(kn), _p(vn), _p(E))
    if r:
        raise OracleError(f"lfo_exact_objective failed: {r}")
    return E[:n]


def bf16_bits_to_f64(a) -> np.ndarray:
    """Exact widening of bf16 bit patterns (uint16) to fp64, for tests' own checks."""
    a = np.asarray(a, np.uint16).astype(np.uint32) << 16
    return a.view(np.float32).astype(np.float64)
