"""Thin ctypes binding of the LongFlow C ABI (include/longflow.h) -- argument marshalling only.

Every step of the decode path runs in liblongflow.so's CUDA kernels; this module converts
Python/torch arguments to plain pointers and sizes and raises on non-LF_OK status.  torch is
used only for device memory and streams.  There is no CPU fallback: if the library is
missing or the device is not a B200 the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblongflow.so")

LF_OK = 0
STATUS = {0: "LF_OK", 1: "LF_ERR_INVALID_ARGUMENT", 2: "LF_ERR_UNSUPPORTED", 3: "LF_ERR_OUT_OF_MEMORY",
          4: "LF_ERR_PREFILL_EXCEEDS_BUDGET", 5: "LF_ERR_CUDA"}
DTYPES = {"bf16": 0, "f32": 1}
KERNELS = {"auto": 0, "simt": 1, "tcgen05": 2}
KERNEL_NAMES = {v: k for k, v in KERNELS.items()}

EXPORTS = ["lf_cache_bytes", "lf_cache_create", "lf_cache_destroy", "lf_prefill_fill", "lf_decode_step",
           "lf_decode_step_host", "lf_cache_views", "lf_cache_plan", "lf_cache_plan_detail", "lf_kernels_per_step",
           "lf_debug_set_trace", "lf_cache_pending", "lf_snapkv_workspace_bytes", "lf_prefill_snapkv",
           "lf_diag_workspace_bytes", "lf_diagnose_step", "lf_status_string", "lf_last_error"]
MODES = {"same_step": 0, "deferred": 1, "deferred_exclude_newest": 2}


class LFError(RuntimeError):
    def __init__(self, status, what, detail):
        super().__init__(f"{what}: {STATUS.get(status, status)}: {detail}")
        self.status = status


class CacheConfig(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("budget", ctypes.c_int32), ("out_dtype", ctypes.c_int32),
                ("softmax_scale", ctypes.c_float), ("mode", ctypes.c_int32), ("kernel", ctypes.c_int32),
                ("split_tokens", ctypes.c_int32), ("plan_batch", ctypes.c_int32), ("seq_offset", ctypes.c_int32),
                ("plan_shards", ctypes.c_int32),
                ("ctas_per_sm", ctypes.c_int32), ("solo", ctypes.c_int32), ("latency_variant", ctypes.c_int32)]


_lib = None


def load(path: str = os.environ.get("LF_LIB", LIB_PATH)):
    """Load liblongflow.so (raises if it has not been built: run __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: the CUDA extension is not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(path)
    P, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
    cfgp = ctypes.POINTER(CacheConfig)
    lib.lf_cache_bytes.argtypes = [cfgp, ctypes.POINTER(sz)]
    lib.lf_cache_create.argtypes = [cfgp, ctypes.c_int, P, sz, ctypes.POINTER(P)]
    lib.lf_cache_destroy.argtypes = [P]
    lib.lf_prefill_fill.argtypes = [P, i32, P, P, i32, P]
    lib.lf_decode_step.argtypes = [P, P, P, P, P, P, P, P]
    lib.lf_decode_step_host.argtypes = [P, P, P, P, P, P, P]
    lib.lf_cache_views.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P)]
    lib.lf_cache_plan.argtypes = [P, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]
    lib.lf_cache_plan_detail.argtypes = [P] + [ctypes.POINTER(i32)] * 6
    lib.lf_cache_plan_detail.restype = ctypes.c_int
    lib.lf_snapkv_workspace_bytes.argtypes = [P, i32, i32, ctypes.POINTER(sz)]
    lib.lf_snapkv_workspace_bytes.restype = ctypes.c_int
    lib.lf_prefill_snapkv.argtypes = [P, i32, P, P, P, i32, i32, i32, P, P, P]
    lib.lf_prefill_snapkv.restype = ctypes.c_int
    lib.lf_diag_workspace_bytes.argtypes = [P, ctypes.POINTER(sz)]
    lib.lf_diag_workspace_bytes.restype = ctypes.c_int
    lib.lf_diagnose_step.argtypes = [P, P, P, P, P, P, P, P]
    lib.lf_diagnose_step.restype = ctypes.c_int
    lib.lf_cache_pending.argtypes = [P, ctypes.POINTER(P)]
    lib.lf_cache_pending.restype = ctypes.c_int
    lib.lf_debug_set_trace.argtypes = [P, P]
    lib.lf_debug_set_trace.restype = ctypes.c_int
    lib.lf_kernels_per_step.argtypes = [P]
    lib.lf_kernels_per_step.restype = i32
    for f in ("lf_cache_bytes", "lf_cache_create", "lf_cache_destroy", "lf_prefill_fill", "lf_decode_step",
              "lf_decode_step_host", "lf_cache_views", "lf_cache_plan"):
        getattr(lib, f).restype = ctypes.c_int
    lib.lf_status_string.argtypes = [ctypes.c_int]
    lib.lf_status_string.restype = ctypes.c_char_p
    lib.lf_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _check(st, what):
    if st != LF_OK:
        raise LFError(st, what, load().lf_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


# plan overrides (lf_cache_config): None/"auto" = automatic
_SOLO = {None: 0, "auto": 0, False: 1, True: 2}
_LAT = {None: 0, "auto": 0, False: 1, True: 2}


def make_config(batch, num_q_heads, num_kv_heads, head_dim, budget, out_dtype="f32", softmax_scale=0.0,
                kernel="auto", split_tokens=0, mode="same_step", plan_batch=0, seq_offset=0, plan_shards=0,
                ctas_per_sm=0, solo=None, latency_variant=None) -> CacheConfig:
    return CacheConfig(batch, num_q_heads, num_kv_heads, head_dim, budget, DTYPES[out_dtype],
                       float(softmax_scale), MODES[mode], KERNELS[kernel], split_tokens, plan_batch, seq_offset,
                       plan_shards, ctas_per_sm, _SOLO[solo], _LAT[latency_variant])


def cache_bytes(cfg: CacheConfig) -> int:
    n = ctypes.c_size_t()
    _check(load().lf_cache_bytes(ctypes.byref(cfg), ctypes.byref(n)), "lf_cache_bytes")
    return n.value


class Cache:
    """A static KV cache on one GPU plus the fused decode step (lf_decode_step).

    By default the slab is a torch uint8 CUDA tensor passed as caller-owned device memory
    (`library_owned=True` makes the library do its single cudaMalloc instead).  A rank's shard of a
    global batch passes plan_batch (the global batch), seq_offset (its first sequence) and plan_shards
    (the number of shards) so every unit is computed exactly as a one-GPU cache of the whole batch with
    the same plan_shards computes it; ctas_per_sm / solo / latency_variant override the plan.
    """

    def __init__(self, batch, num_q_heads, num_kv_heads, head_dim, budget, out_dtype="f32",
                 softmax_scale=0.0, kernel="auto", split_tokens=0, device=0, library_owned=False,
                 mode="same_step", plan_batch=0, seq_offset=0, plan_shards=0, ctas_per_sm=0, solo=None,
                 latency_variant=None):
        lib = load()
        self.cfg = make_config(batch, num_q_heads, num_kv_heads, head_dim, budget, out_dtype, softmax_scale,
                               kernel, split_tokens, mode, plan_batch, seq_offset, plan_shards, ctas_per_sm, solo,
                               latency_variant)
        self.B, self.Hq, self.Hkv, self.d, self.N = batch, num_q_heads, num_kv_heads, head_dim, budget
        self.G = num_q_heads // num_kv_heads
        self.out_dtype = out_dtype
        self.device = torch.device("cuda", device)
        self._buf = None
        h = ctypes.c_void_p()
        if library_owned:
            _check(lib.lf_cache_create(ctypes.byref(self.cfg), device, None, 0, ctypes.byref(h)), "lf_cache_create")
        else:
            nbytes = cache_bytes(self.cfg)
            self._buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            _check(lib.lf_cache_create(ctypes.byref(self.cfg), device, self._buf.data_ptr(), nbytes,
                                       ctypes.byref(h)), "lf_cache_create")
        self._h = h

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _check(load().lf_cache_destroy(self._h), "lf_cache_destroy")
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- calls
    def prefill(self, seq, k, v, stream=None):
        """k, v: bf16 CUDA tensors [Hkv][n][d]."""
        n = 0 if k is None else int(k.shape[1])
        _check(load().lf_prefill_fill(self._h, seq, _ptr(k), _ptr(v), n, _stream(stream)), "lf_prefill_fill")

    def prefill_snapkv(self, seq, k, v, q_obs, window=32, pool_kernel=7, kept=None, stream=None):
        """SnapKV-compressed prefill (NEXT-f3): k, v bf16 [Hkv][n][d], q_obs bf16 [Hq][w][d]."""
        n, w = int(k.shape[1]), int(window)
        nb = ctypes.c_size_t()
        _check(load().lf_snapkv_workspace_bytes(self._h, n, w, ctypes.byref(nb)), "lf_snapkv_workspace_bytes")
        ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=self.device)
        _check(load().lf_prefill_snapkv(self._h, seq, _ptr(k), _ptr(v), _ptr(q_obs), n, w, pool_kernel, _ptr(kept),
                                        ws.data_ptr(), _stream(stream)), "lf_prefill_snapkv")
        return ws   # keep alive until the stream has run it

    def diagnose_step(self, q, k_new, v_new, stream=None):
        """NEXT-f4 diagnostics on the pre-step cache: (islot int32 [B][Hkv][3], fstat fp32 [B][Hkv][3])."""
        nb = ctypes.c_size_t()
        _check(load().lf_diag_workspace_bytes(self._h, ctypes.byref(nb)), "lf_diag_workspace_bytes")
        ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=self.device)
        islot = torch.empty(self.B, self.Hkv, 3, dtype=torch.int32, device=self.device)
        fstat = torch.empty(self.B, self.Hkv, 3, dtype=torch.float32, device=self.device)
        _check(load().lf_diagnose_step(self._h, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(islot), _ptr(fstat),
                                       ws.data_ptr(), _stream(stream)), "lf_diagnose_step")
        self._diag_ws = ws
        return islot, fstat

    def decode_step(self, q, k_new, v_new, out, slot, scores=None, stream=None):
        _check(load().lf_decode_step(self._h, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out), _ptr(slot),
                                     _ptr(scores), _stream(stream)), "lf_decode_step")

    def decode_step_host(self, q, k_new, v_new, out, slot, stream=None):
        """Host (preferably pinned) torch tensors in, host tensors out (synchronous)."""
        _check(load().lf_decode_step_host(self._h, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out), _ptr(slot),
                                          _stream(stream)), "lf_decode_step_host")

    # -- introspection
    def raw_views(self):
        k, v, nv = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(load().lf_cache_views(self._h, ctypes.byref(k), ctypes.byref(v), ctypes.byref(nv)), "views")
        return k.value, v.value, nv.value

    def views(self):
        """(K, V bf16 [B][Hkv][N][d], n_valid int32 [B][Hkv]) as torch views of the slab
        (only for the default caller-owned slab)."""
        if self._buf is None:
            raise RuntimeError("views() needs the caller-owned slab")
        kp, vp, nvp = self.raw_views()
        base = self._buf.data_ptr()
        kv = self.B * self.Hkv * self.N * self.d * 2

        def sl(p, nbytes):
            return self._buf[p - base:p - base + nbytes]
        K = sl(kp, kv).view(torch.bfloat16).view(self.B, self.Hkv, self.N, self.d)
        V = sl(vp, kv).view(torch.bfloat16).view(self.B, self.Hkv, self.N, self.d)
        nv = sl(nvp, self.B * self.Hkv * 4).view(torch.int32).view(self.B, self.Hkv)
        return K, V, nv

    def pending(self):
        """Deferred modes: int32 [B][Hkv] torch view of the slot the next token will cover."""
        pp = ctypes.c_void_p()
        _check(load().lf_cache_pending(self._h, ctypes.byref(pp)), "lf_cache_pending")
        base = self._buf.data_ptr()
        return self._buf[pp.value - base:pp.value - base + self.B * self.Hkv * 4].view(torch.int32).view(
            self.B, self.Hkv)

    def plan(self):
        k, s, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(load().lf_cache_plan(self._h, ctypes.byref(k), ctypes.byref(s), ctypes.byref(c)), "plan")
        cl, st, tc, sm, so, lt = (ctypes.c_int32() for _ in range(6))
        _check(load().lf_cache_plan_detail(self._h, ctypes.byref(cl), ctypes.byref(st), ctypes.byref(tc),
                                           ctypes.byref(sm), ctypes.byref(so), ctypes.byref(lt)), "plan_detail")
        return dict(kernel=KERNEL_NAMES[k.value], splits=s.value, split_tokens=c.value, clusters=cl.value,
                    stages=st.value, tmem_cols=tc.value, smem=sm.value, solo_rounds=so.value,
                    latency_variant=lt.value)

    def set_trace(self, buf):
        """Debug: device buffer for the -DLF_TRACE event trace (None disables)."""
        _check(load().lf_debug_set_trace(self._h, _ptr(buf)), "lf_debug_set_trace")

    def kernels_per_step(self) -> int:
        return int(load().lf_kernels_per_step(self._h))

    # -- allocation helpers for outputs (torch device memory only)
    def new_outputs(self, with_scores=False):
        dt = torch.float32 if self.out_dtype == "f32" else torch.bfloat16
        out = torch.empty(self.B, self.Hq, self.d, dtype=dt, device=self.device)
        slot = torch.empty(self.B, self.Hkv, dtype=torch.int32, device=self.device)
        scores = (torch.empty(self.B, self.Hkv, self.N, dtype=torch.float32, device=self.device)
                  if with_scores else None)
        return out, slot, scores
