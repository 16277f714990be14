"""Seeded synthetic inputs for the LongFlow decode step (shared by tests, smoke and bench).

This module holds NO arithmetic of the method (no logits, softmax, scores or argmin):
only the workload shapes of BASELINE.json and the random draws that feed both the CUDA
path and the oracle.  Recipe:

* queries  -- per (sequence, query head) a unit-sphere random walk
             u_{t+1} = normalize(0.95 u_t + 0.05 g_t), g_t a unit Gaussian direction
             (adjacent cosine ~0.9986, the "high and stable similarity between adjacent
             queries" of P:105 / P:626); q = sigma_s * sqrt(d) * u, so q.k/sqrt(d) ~ N(0, sigma_s^2)
* keys     -- N(0, 1), optionally times per-(kv head, channel) scales exp(0.5 N(0,1)) (outlier channels)
* values   -- N(0, 1)
* prefill  -- iid rows from the same distributions; every decode step draws fresh (q, k*, v*)
* rounding -- everything is rounded to bf16 (round-to-nearest-even) at generation

All tensors are torch bf16; ``bits()`` gives the uint16 bit patterns the oracle takes.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch


@dataclasses.dataclass(frozen=True)
class Workload:
    tag: str
    B: int
    Hq: int
    Hkv: int
    d: int
    N: int            # budget (static slots per sequence and kv head)
    prefill: int      # prompt tokens loaded before decoding
    steps: int        # decode steps of the paper-shaped run (T = prefill + steps)
    note: str = ""

    @property
    def G(self) -> int:
        return self.Hq // self.Hkv

    @property
    def units(self) -> int:
        return self.B * self.Hkv


# BASELINE.json configs -> concrete shapes.
CONFIGS = {
    "tiny": Workload("tiny", 1, 1, 1, 64, 128, 16, 512,
                     "configs[0]: batch=1, 1 kv / 1 q head, d=64, budget 128, 512 decode steps"),
    "q7": Workload("q7", 1, 28, 4, 128, 2048, 512, 9728,
                   "configs[1]: single sequence Qwen-7B-like GQA 28/4, d=128, budget 2048, 10k gen (80% compression)"),
    "q3": Workload("q3", 64, 32, 8, 128, 4096, 512, 32768,
                   "configs[2]: batch=64 Qwen3-8B-like GQA 32/8, d=128, budget 4096, 32k decode"),
    "r": Workload("r", 256, 32, 8, 128, 8192, 512, 40448,
                  "configs[3]: batch=256 long-output decode, budget 8192 (32/8 GQA assumed), sharded by sequence"),
    "f1": Workload("f1", 128, 32, 8, 128, 3200, 512, 16000,
                   "paper Fig. 1 shape (P:45): Qwen3-8B, batch 128, cache 3200 (context only)"),
}


def sweep_workload(B: int, N: int) -> Workload:
    """configs[4]: budget sweep point at fixed 80% compression (T = 5N), 32/8 GQA, d=128."""
    pre = min(512, N // 2)
    return Workload(f"sweep_b{B}_n{N}", B, 32, 8, 128, N, pre, 5 * N - pre)


def bits(t: torch.Tensor) -> np.ndarray:
    """bf16 tensor -> uint16 numpy array of its bit patterns (host copy)."""
    assert t.dtype == torch.bfloat16
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def from_bits(a: np.ndarray, device="cpu") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, np.uint16).view(np.int16)).view(torch.bfloat16).to(device)


def bf16(x, device="cpu") -> torch.Tensor:
    """Round values (exact fixtures or floats) to bf16, RNE."""
    return torch.as_tensor(np.asarray(x, np.float64), dtype=torch.float64).to(torch.float32).to(
        torch.bfloat16).to(device)


def _gen(seed: int, stream: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1_000_003 + int(stream) * 7919 + 17) % (2**63 - 1))
    return g


class Synth:
    """Deterministic generator for one workload: prefill rows and per-step (q, k*, v*).

    sigma_s: logit scale (default 2; SURVEY D.2 sweep {1, 2, 4}, stress 12).
    key_outliers: per-(kv head, channel) key scales exp(0.5 N(0,1)).
    """

    def __init__(self, wl: Workload, seed: int = 0, device="cpu", sigma_s: float = 2.0,
                 key_outliers: bool = False, B: int | None = None, b0: int = 0):
        self.wl = wl
        self.seed = seed
        self.device = torch.device(device)
        self.sigma_s = float(sigma_s)
        # a shard [b0, b0+B) of the batch draws exactly the rows the full batch would
        self.B = wl.B if B is None else B
        self.b0 = b0
        d = wl.d
        g = _gen(seed, 1, self.device)
        self.key_scale = None
        if key_outliers:
            self.key_scale = torch.exp(0.5 * torch.randn(wl.Hkv, d, generator=g, device=self.device))
        # initial query directions, one generator per sequence (sharding-stable)
        u = _per_seq(seed, 4, (wl.Hq, d), b0, self.B, self.device, torch.float32)
        self.u = torch.nn.functional.normalize(u, dim=-1).contiguous()
        self.t = 0

    def _rows(self, stream: int, shape_full, dtype=torch.float32):
        """Rows of sequences [b0, b0+B): each sequence has its own generator, so a shard
        draws exactly the rows the full batch would (multi-GPU bit-identity)."""
        return _per_seq(self.seed, stream, shape_full[1:], self.b0, self.B, self.device, dtype)

    def prefill(self, n: int | None = None):
        """K, V bf16 [B][Hkv][n][d] (n defaults to the workload's prefill length)."""
        wl = self.wl
        n = wl.prefill if n is None else n
        k = self._rows(2, (wl.B, wl.Hkv, n, wl.d))
        if self.key_scale is not None:
            k = k * self.key_scale[None, :, None, :]
        v = self._rows(3, (wl.B, wl.Hkv, n, wl.d))
        return k.to(torch.bfloat16).contiguous(), v.to(torch.bfloat16).contiguous()

    def step(self):
        """Next decode step's q [B][Hq][d], k_new, v_new [B][Hkv][d], all bf16."""
        wl = self.wl
        t = self.t
        self.t += 1
        gdir = torch.nn.functional.normalize(self._rows(1000 + 3 * t, (wl.B, wl.Hq, wl.d)), dim=-1)
        self.u = torch.nn.functional.normalize(0.95 * self.u + 0.05 * gdir, dim=-1)
        q = (self.sigma_s * math.sqrt(wl.d)) * self.u
        k = self._rows(1001 + 3 * t, (wl.B, wl.Hkv, wl.d))
        if self.key_scale is not None:
            k = k * self.key_scale[None, :, :]
        v = self._rows(1002 + 3 * t, (wl.B, wl.Hkv, wl.d))
        return (q.to(torch.bfloat16).contiguous(), k.to(torch.bfloat16).contiguous(),
                v.to(torch.bfloat16).contiguous())


def _per_seq(seed, stream, shape, b0, B, device, dtype=torch.float32):
    out = torch.empty((B, *shape), device=device, dtype=dtype)
    for i in range(B):
        g = _gen(seed, stream * 1_048_576 + b0 + i, device)
        out[i] = torch.randn(*shape, generator=g, device=device, dtype=dtype)
    return out


def random_cache(B, Hkv, N, d, seed=0, device="cpu", b0=0):
    """Full random K, V bf16 [B][Hkv][N][d] for sequences [b0, b0+B) (steady-state bench
    caches, every slot valid): N(0,1) rows, one generator per sequence."""
    k = torch.empty(B, Hkv, N, d, device=device, dtype=torch.bfloat16)
    v = torch.empty_like(k)
    for i in range(B):
        g = _gen(seed, 77 * 1_048_576 + b0 + i, device)
        k[i] = torch.randn(Hkv, N, d, generator=g, device=device).to(torch.bfloat16)
        v[i] = torch.randn(Hkv, N, d, generator=g, device=device).to(torch.bfloat16)
    return k, v
