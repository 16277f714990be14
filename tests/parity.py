"""Shared GPU-vs-oracle parity machinery (tests only).

Tolerances (reading R12, from BASELINE.json north_star):
  out     fp32-out mode: normwise per (sequence, q head) row, max_l|o - o^| / max_l|o^| <= 2e-3
          bf16-out mode: every element is the single RNE rounding of a value within 1e-4 x max|o^_row|
          of o^: |o_bf16 - o^| <= ulp(o_bf16)/2 + ulp(o^)/2 + 1e-4 max|o^_row| (elementwise)
  scores  |I - I^| <= 1e-4 I^ + 1e-30 elementwise on valid slots; +inf on invalid slots
  slot    identical, except an accepted near-tie: I^_slot <= (1 + 1e-4) min_k I^_k + 1e-30;
          then the oracle adopts the GPU's slot (both are correct, R13) so the two caches stay
          bit-identical.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

import oracle
from lf_synth import Synth, Workload, bits

OUT_TOL = 2e-3
BF16_FP32_SLACK = 1e-4   # bf16 out: fp32-path error allowed before the single rounding (R12)
SCORE_RTOL = 1e-4
SCORE_ATOL = 1e-30


@dataclasses.dataclass
class Stats:
    steps: int = 0
    max_out_err: float = 0.0
    max_score_err: float = 0.0
    adoptions: int = 0
    evictions: int = 0
    bf16_exact_frac: float = 1.0   # bf16 out: fraction of elements equal to RNE(oracle)


def bf16_ulp(x: np.ndarray) -> np.ndarray:
    ax = np.abs(x).astype(np.float64)
    e = np.floor(np.log2(np.maximum(ax, 2.0 ** -126)))
    return 2.0 ** (e - 7)


def check_out(o_gpu: np.ndarray, o_ref: np.ndarray, out_dtype: str, stats: Stats):
    if out_dtype == "f32":
        den = np.abs(o_ref).max(axis=-1)
        num = np.abs(o_gpu - o_ref).max(axis=-1)
        err = np.where(den > 0, num / np.maximum(den, 1e-300), num)
        stats.max_out_err = max(stats.max_out_err, float(err.max()))
        assert err.max() <= OUT_TOL, f"out normwise error {err.max():.3e} > {OUT_TOL}"
    else:
        # bf16 out = RNE of the kernel's fp32 result, rounded ONCE: each element must equal the bf16
        # rounding of some value within BF16_FP32_SLACK * max|o^_row| of the exact o^ (R12):
        #   |o_bf16 - o^| <= ulp(o_bf16)/2 + ulp(o^)/2 + slack * max|o^_row|
        # i.e. RNE(o^) or its neighbour where o^ sits within the fp32 error of a rounding boundary,
        # and an absolute fp32-size allowance for elements near zero (their ulp is tiny).
        den = np.abs(o_ref).max(axis=-1, keepdims=True)
        excess = np.abs(o_gpu - o_ref) - 0.5 * bf16_ulp(o_gpu) - 0.5 * bf16_ulp(o_ref)
        rel = np.maximum(excess, 0.0) / np.maximum(den, 1e-300)
        stats.max_out_err = max(stats.max_out_err, float(rel.max()))
        bad = rel > BF16_FP32_SLACK
        assert not bad.any(), (f"bf16 out: not a single rounding of a value within {BF16_FP32_SLACK} (normwise) "
                               f"of the exact output at {np.argwhere(bad)[:5]} (excess {rel.max():.3e})")
        ref_bf16 = torch.from_numpy(o_ref).to(torch.float32).to(torch.bfloat16).double().numpy()
        stats.bf16_exact_frac = float((o_gpu == ref_bf16).mean())


def check_scores(sc_gpu: np.ndarray, sc_ref: np.ndarray, n_valid: np.ndarray, stats: Stats):
    B, H, N = sc_ref.shape
    for b in range(B):
        for h in range(H):
            n = int(n_valid[b, h])
            g, r = sc_gpu[b, h, :n].astype(np.float64), sc_ref[b, h, :n]
            err = np.abs(g - r)
            bad = err > SCORE_RTOL * r + SCORE_ATOL
            if n:
                rel = err / np.maximum(r, 1e-300)
                stats.max_score_err = max(stats.max_score_err, float(np.where(r > 1e-30, rel, 0).max()))
            assert not bad.any(), (f"score mismatch unit ({b},{h}) slots {np.nonzero(bad)[0][:5]}: "
                                   f"gpu {g[bad][:3]} ref {r[bad][:3]}")
            assert np.all(np.isinf(sc_gpu[b, h, n:])), f"unit ({b},{h}): invalid slots must score +inf"


def accept_slots(slot_gpu: np.ndarray, slot_ref: np.ndarray, sc_ref: np.ndarray, n_valid: np.ndarray,
                 N: int, stats: Stats) -> np.ndarray:
    """Returns the slots the oracle commits: its own, or the GPU's at an accepted near-tie."""
    chosen = slot_ref.copy()
    for u in np.ndindex(slot_ref.shape):
        n = int(n_valid[u])
        if n < N:
            assert slot_gpu[u] == n, f"unit {u}: append slot {slot_gpu[u]} != n {n}"
            continue
        stats.evictions += 1
        if slot_gpu[u] == slot_ref[u]:
            continue
        s = int(slot_gpu[u])
        assert 0 <= s < n, f"unit {u}: slot {s} out of range"
        m = sc_ref[u][:n].min()
        assert sc_ref[u][s] <= (1 + SCORE_RTOL) * m + SCORE_ATOL, (
            f"unit {u}: GPU slot {s} (I={sc_ref[u][s]:.6e}) vs oracle slot {slot_ref[u]} (I={m:.6e})")
        chosen[u] = s
        stats.adoptions += 1
    return chosen


def run_lockstep(cache, orc: oracle.OracleCache, syn: Synth, steps: int, out_dtype="f32",
                 with_scores=True, check_cache_every=0) -> Stats:
    """Drive the CUDA path and the oracle on the same seeded bf16 inputs, comparing every step."""
    st = Stats()
    out, slot, scores = cache.new_outputs(with_scores=with_scores)
    dev = cache.device
    for t in range(steps):
        q, kn, vn = syn.step()
        nv_before = orc.n_valid.copy()
        cache.decode_step(q.to(dev), kn.to(dev), vn.to(dev), out, slot, scores)
        torch.cuda.synchronize()
        qb, kb, vb = bits(q), bits(kn), bits(vn)
        o_ref, s_ref, sc_ref = orc.compute(qb, kb, vb, want_scores=True)
        check_out(out.cpu().double().numpy(), o_ref, out_dtype, st)
        if with_scores:
            check_scores(scores.cpu().numpy(), sc_ref, nv_before, st)
        chosen = accept_slots(slot.cpu().numpy(), s_ref, sc_ref, nv_before, orc.N, st)
        orc.apply(kb, vb, chosen)
        st.steps += 1
        if check_cache_every and (t + 1) % check_cache_every == 0:
            assert_cache_equal(cache, orc)
    assert_cache_equal(cache, orc)
    return st


def assert_cache_equal(cache, orc: oracle.OracleCache):
    K, V, nv = cache.views()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(nv.cpu().numpy(), orc.n_valid)
    np.testing.assert_array_equal(bits(K), orc.K)
    np.testing.assert_array_equal(bits(V), orc.V)


def setup_pair(wl: Workload, kernel="auto", out_dtype="f32", seed=0, prefill=None, split_tokens=0,
               sigma_s=2.0, scale=0.0, nthreads=4, key_outliers=False, **plan_kw):
    """(cache, oracle, synth) on the same seeded inputs; plan_kw: ctas_per_sm / solo /
    latency_variant overrides of the split plan."""
    from paper_2603_11504_b200 import Cache
    syn = Synth(wl, seed=seed, sigma_s=sigma_s, key_outliers=key_outliers)
    cache = Cache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N, out_dtype=out_dtype, kernel=kernel,
                  split_tokens=split_tokens, softmax_scale=scale, **plan_kw)
    orc = oracle.OracleCache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N, scale=scale or None, nthreads=nthreads)
    n = wl.prefill if prefill is None else prefill
    if n > 0:
        K, V = syn.prefill(n)
        for b in range(wl.B):
            cache.prefill(b, K[b].cuda(), V[b].cuda())
            orc.prefill(b, bits(K[b]), bits(V[b]))
    return cache, orc, syn
