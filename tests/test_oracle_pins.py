"""Pins for the fp64 oracle (oracle/lfo.c) against what the paper and mathematics fix.

Each test names the passage it follows (P:n = PAPER.md line n, S:n = SPEC.md line n,
C.3 #k = SURVEY.md section 8(c) pin table).  None of these tests calls the CUDA path.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from lf_synth import CONFIGS, Synth, bits, bf16

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _b(x):
    """exact values -> bf16 bit patterns (uint16)."""
    return bits(bf16(x))


def _f64(u16):
    return oracle.bf16_bits_to_f64(u16)


def _scale(s):
    return {"ln2": math.log(2.0), "ln3": math.log(3.0)}.get(s, s)


def _rand_unit(rng, G, d, n, qs=1.0):
    q = _b(rng.standard_normal((G, d)) * qs)
    K = _b(rng.standard_normal((n, d)))
    V = _b(rng.standard_normal((n, d)))
    return q, K, V


# --- softmax / weights -------------------------------------------------------------

def test_softmax_closed_forms():
    """S:46-48 (Eq. 1): [ln1, ln3] -> [1/4, 3/4]; [0,0] -> [1/2,1/2]; single support -> 1."""
    gold = json.load(open(os.path.join(GOLD, "softmax_closed_forms.json")))
    for case in gold["cases"]:
        keys = np.array(case["keys"], np.float64)[:, None]
        r = oracle.unit_attend(_b([[1.0]]), _b(keys), _b(np.zeros_like(keys)), scale=_scale(case["scale"]))
        np.testing.assert_allclose(r["alpha"][0], case["alpha"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("n", [1, 7, 1000, 10000])
def test_softmax_sums_to_one(n):
    """Invariant of Eq. 1: sum_j alpha_j = 1 within 1e-12 for logits in [-50, 50]."""
    rng = np.random.default_rng(n)
    keys = _b(rng.uniform(-50, 50, size=(n, 1)))
    r = oracle.unit_attend(_b([[1.0]]), keys, _b(rng.standard_normal((n, 1))), scale=1.0)
    assert abs(r["alpha"].sum() - 1.0) < 1e-12
    assert np.all(r["alpha"] >= 0)
    # with the new token attended the weights over n+1 tokens also sum to one (Eq. 4 Z)
    r2 = oracle.unit_attend(_b([[1.0]]), keys, _b(rng.standard_normal((n, 1))),
                            _b([3.0]), _b([1.0]), scale=1.0)
    assert abs(r2["alpha"].sum() - 1.0) < 1e-12


def test_large_logits_no_overflow():
    """R5 / P:205: dropping the running max overflows fp32 at s > 88.7; the exact-max oracle
    must stay finite for a logit range of ~100 (SURVEY D.2 stress sigma_s = 12)."""
    rng = np.random.default_rng(5)
    q = _b(rng.standard_normal((4, 128)) * 12.0)
    K = _b(rng.standard_normal((512, 128)))
    V = _b(rng.standard_normal((512, 128)))
    r = oracle.unit_attend(q, K, V, K[0], V[0])
    assert np.all(np.isfinite(r["out"])) and np.all(np.isfinite(r["scores"]))
    assert np.allclose(r["alpha"].sum(axis=1), 1.0, atol=1e-12)


# --- attention output ----------------------------------------------------------------

def test_single_support_output_is_v():
    """a single valid token gets weight 1, so o = v."""
    rng = np.random.default_rng(1)
    q, K, V = _rand_unit(rng, 3, 16, 1)
    r = oracle.unit_attend(q, K, V)
    np.testing.assert_array_equal(r["out"], np.repeat(_f64(V), 3, axis=0))


def test_orthogonal_query_gives_mean():
    """q orthogonal to every key -> uniform weights -> o = mean(v)."""
    K = _b([[0.0, 1.0], [0.0, -2.0], [0.0, 0.5], [0.0, 3.0]])
    V = _b([[1.0, 2.0], [3.0, -4.0], [0.5, 0.25], [-2.0, 8.0]])
    r = oracle.unit_attend(_b([[1.0, 0.0]]), K, V)
    np.testing.assert_allclose(r["out"][0], _f64(V).mean(axis=0), rtol=0, atol=1e-15)


@pytest.mark.parametrize("G,d,n", [(1, 8, 5), (4, 64, 33), (7, 128, 129), (2, 3, 1)])
def test_matches_torch_sdpa_fp64(G, d, n):
    """C.3 #4: Eq. 1 through an independent library route (torch fp64 SDPA), new token attended."""
    rng = np.random.default_rng(G * 1000 + n)
    q, K, V = _rand_unit(rng, G, d, n, qs=2.0)
    kn, vn = _b(rng.standard_normal(d)), _b(rng.standard_normal(d))
    r = oracle.unit_attend(q, K, V, kn, vn)
    Kall = torch.from_numpy(np.vstack([_f64(K), _f64(kn)[None]]))
    Vall = torch.from_numpy(np.vstack([_f64(V), _f64(vn)[None]]))
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(_f64(q))[None, :, None, :], Kall[None, None].expand(1, G, -1, -1),
        Vall[None, None].expand(1, G, -1, -1))[0, :, 0, :].numpy()
    np.testing.assert_allclose(r["out"], ref, rtol=1e-12, atol=1e-13)


# --- LongFlowScore -------------------------------------------------------------------

@pytest.mark.parametrize("G,d,n", [(1, 16, 9), (4, 64, 40), (7, 32, 17)])
def test_scores_brute_force_contribution_vectors(G, d, n):
    """C.3 #5: materialise alpha (torch fp64 softmax), the contribution vectors C_j = P_j V_j
    (Alg. 1, Eq. 5), their row L1 normalised once, then the
    mean over the group (R2).  Also sum_j c_j + c_* = o (Eq. 5 decomposition)."""
    rng = np.random.default_rng(n)
    q, K, V = _rand_unit(rng, G, d, n, qs=2.0)
    kn, vn = _b(rng.standard_normal(d)), _b(rng.standard_normal(d))
    r = oracle.unit_attend(q, K, V, kn, vn)
    Qf = torch.from_numpy(_f64(q))
    Kf = torch.from_numpy(np.vstack([_f64(K), _f64(kn)[None]]))
    Vf = torch.from_numpy(np.vstack([_f64(V), _f64(vn)[None]]))
    alpha = torch.softmax(Qf @ Kf.T / math.sqrt(d), dim=-1)            # [G][n+1]
    C = alpha[:, :, None] * Vf[None, :, :]                            # [G][n+1][d]
    per_head = C.abs().sum(dim=-1)[:, :n]                             # [G][n]
    brute = per_head.mean(dim=0).numpy()
    np.testing.assert_allclose(r["scores"], brute, rtol=1e-12, atol=0)
    np.testing.assert_allclose(C.sum(dim=1).numpy(), r["out"], rtol=1e-12, atol=1e-14)
    assert r["slot"] == int(np.argmin(brute))


def test_spec_d1_worked_example_and_appendix_a():
    """S:205-206, S:224, S:279 (Eq. 1 / Eq. 6) and S:353-371 (App. A remainder)."""
    g = json.load(open(os.path.join(GOLD, "spec_d1_example.json")))
    sc = _scale(g["scale"])
    q, K, V = _b(g["q"]), _b(g["K"]), _b(g["V"])
    r = oracle.unit_attend(q, K, V, scale=sc)
    np.testing.assert_allclose(r["alpha"][0], g["alpha"], atol=1e-15)
    np.testing.assert_allclose(r["out"][0, 0], g["out"], atol=1e-15)
    np.testing.assert_allclose(r["scores"], g["scores"], atol=1e-15)
    assert r["slot"] == g["slot"]
    # exact output change when evicting token i (Eq. 4): re-run attention without row i
    for i, want in enumerate(g["delta_o_all"]):
        keep = [j for j in range(2) if j != i]
        ri = oracle.unit_attend(q, K[keep], V[keep], scale=sc)
        assert abs(abs(r["out"][0, 0] - ri["out"][0, 0]) - want) < 1e-15
    r0 = oracle.unit_attend(q, K[[1]], V[[1]], scale=sc)
    delta = r["out"][0, 0] - r0["out"][0, 0]
    a0 = r["alpha"][0, 0]
    c0 = a0 * _f64(V)[0, 0]
    R_closed = -a0 / (1 - a0) * (r["out"][0, 0] - c0)
    assert abs(delta - g["delta_o_evict0"]) < 1e-15
    assert abs(c0 - g["contribution_0"]) < 1e-15
    assert abs((delta - c0) - g["remainder_0"]) < 1e-15 and abs(R_closed - g["remainder_0"]) < 1e-15
    Vmax = np.abs(_f64(V)).max()
    assert abs(2 * Vmax * a0 / (1 - a0) - g["remainder_bound_0"]) < 1e-15


def test_exact_objective_d1_worked_example():
    """NEXT-f4 oracle (brute-force re-attention, Eq. 3's right-hand side P:110) on the d=1 worked
    example: ||o - o^(-i)||^2 = (0.75^2, 2.25^2) (the exact output changes), argmin 0 like the
    LongFlow score."""
    g = json.load(open(os.path.join(GOLD, "spec_d1_example.json")))
    sc = _scale(g["scale"])
    E = oracle.exact_objective(_b(g["q"]), _b(g["K"]), _b(g["V"]), scale=sc)
    np.testing.assert_allclose(E, np.square(g["delta_o_all"]), rtol=0, atol=1e-14)
    assert int(np.argmin(E)) == g["slot"]


@pytest.mark.parametrize("G,d,n", [(1, 16, 9), (4, 32, 40), (7, 64, 25)])
def test_exact_objective_matches_appendix_a_closed_form(G, d, n):
    """The brute-force objective equals App. A's exact change (Delta o = alpha/(1-alpha)
    (v_i - o), so ||Delta o||^2 = (alpha/(1-alpha))^2 ||v_i - o||^2), mean over the group (R25), on
    random units with the current token attended -- two independent routes to the same number."""
    rng = np.random.default_rng(G * 1000 + n)
    q, K, V = _b(rng.standard_normal((G, d))), _b(rng.standard_normal((n, d))), _b(rng.standard_normal((n, d)))
    kn, vn = _b(rng.standard_normal(d)), _b(rng.standard_normal(d))
    E = oracle.exact_objective(q, K, V, kn, vn)
    r = oracle.unit_attend(q, K, V, kn, vn)
    a = r["alpha"][:, :n]
    closed = ((a / (1 - a)) ** 2 * ((_f64(V)[None, :, :] - r["out"][:, None, :]) ** 2).sum(-1)).mean(0)
    np.testing.assert_allclose(E, closed, rtol=1e-9, atol=1e-15)


def test_gqa_worked_example():
    """C.3 #7: mean-over-group aggregation evicts slot 2 (max -> 1, head-0 only -> 0)."""
    g = json.load(open(os.path.join(GOLD, "gqa_worked_example.json")))
    sc = _scale(g["scale"])
    q, K, V, kn, vn = _b(g["q"]), _b(g["K"]), _b(g["V"]), _b(g["k_new"]), _b(g["v_new"])
    r = oracle.unit_attend(q, K, V, kn, vn, scale=sc)
    np.testing.assert_allclose(r["alpha"], g["alpha"], atol=1e-15)
    np.testing.assert_allclose(r["out"], g["out"], atol=1e-15)
    np.testing.assert_allclose(r["scores"], g["scores"], atol=1e-15)
    assert r["slot"] == g["slot"]
    per_head = r["alpha"][:, :3] * np.abs(_f64(V)).sum(axis=1)[None]
    np.testing.assert_allclose(per_head, g["per_head_scores"], atol=1e-15)
    assert int(np.argmin(per_head.max(axis=0))) == g["slot_if_max_aggregation"]
    assert int(np.argmin(per_head[0])) == g["slot_if_head0_only"]
    # full same-step protocol through the cache driver: the new token overwrites slot 2
    c = oracle.OracleCache(1, 2, 1, 2, 3, scale=sc)
    c.prefill(0, K[None], V[None])
    out, slot, scores = c.step(q[None], kn[None, None], vn[None, None])
    assert slot[0, 0] == 2
    np.testing.assert_allclose(out[0], g["out"], atol=1e-15)
    np.testing.assert_array_equal(c.K[0, 0], _b(g["K_after"]))
    np.testing.assert_array_equal(c.V[0, 0], _b(g["V_after"]))


def test_tie_rules():
    """C.3 #8: all-zero V -> all scores 0 -> slot 0; duplicate tokens -> lower index."""
    rng = np.random.default_rng(2)
    q, K, _ = _rand_unit(rng, 2, 8, 10)
    r = oracle.unit_attend(q, K, _b(np.zeros((10, 8))))
    assert np.all(r["scores"] == 0) and r["slot"] == 0
    V = _b(rng.standard_normal((10, 8)) * 4)
    K2, V2 = K.copy(), V.copy()
    K2[3] = K2[7] = _b(np.full(8, 0.5))
    V2[3] = V2[7] = _b(np.full(8, 1e-3))     # tiny values: these two are the minimum
    r = oracle.unit_attend(q, K2, V2)
    assert r["scores"][3] == r["scores"][7] and r["slot"] == 3


def test_zero_weight_token_always_evicted():
    """C.3 #9: one token with alpha < 1e-9, all others > 1e-3 -> always evicted."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        n, d = 64, 16
        q = _b(np.ones((1, d)))
        K = _b(rng.uniform(-0.5, 0.5, (n, d)))
        V = _b(rng.standard_normal((n, d)))
        victim = int(rng.integers(n))
        K[victim] = _b(np.full(d, -8.0))
        r = oracle.unit_attend(q, K, V, scale=0.25)
        a = r["alpha"][0]
        assert a[victim] < 1e-9 and np.all(np.delete(a, victim) > 1e-3)
        assert r["slot"] == victim


def test_value_scale_invariance():
    """C.3 #10: V -> 2V (bf16-exact) leaves the slot unchanged and doubles the scores."""
    rng = np.random.default_rng(4)
    q, K, V = _rand_unit(rng, 4, 32, 50)
    r1 = oracle.unit_attend(q, K, V)
    r2 = oracle.unit_attend(q, K, _b(_f64(V) * 2.0))
    assert r1["slot"] == r2["slot"]
    np.testing.assert_allclose(r2["scores"], 2 * r1["scores"], rtol=1e-14)


def test_permutation_equivariance():
    """C.3 #11: permuting slots permutes scores and slot; o is unchanged."""
    rng = np.random.default_rng(6)
    q, K, V = _rand_unit(rng, 4, 32, 50, qs=2.0)
    perm = rng.permutation(50)
    r1 = oracle.unit_attend(q, K, V, K[0], V[0])
    r2 = oracle.unit_attend(q, K[perm], V[perm], K[0], V[0])
    np.testing.assert_allclose(r2["out"], r1["out"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(r2["scores"], r1["scores"][perm], rtol=1e-12)
    assert perm[r2["slot"]] == r1["slot"]


def test_group_replication_reduces_to_single_head():
    """C.3 #12: G identical query heads -> mean-aggregated I equals single-head Eq. 6."""
    rng = np.random.default_rng(7)
    q1, K, V = _rand_unit(rng, 1, 64, 77, qs=2.0)
    r1 = oracle.unit_attend(q1, K, V, K[3], V[5])
    r4 = oracle.unit_attend(np.repeat(q1, 4, axis=0), K, V, K[3], V[5])
    np.testing.assert_allclose(r4["scores"], r1["scores"], rtol=1e-14)
    assert r4["slot"] == r1["slot"]


@pytest.mark.parametrize("seed", range(5))
def test_appendix_a_identities(seed):
    """C.3 #13: exact Delta o_i = c_i + R_i with R_i = -a_i/(1-a_i)(o - c_i),
    ||R_i|| <= 2 V a_i/(1-a_i), and renormalised weights a_j^(\\i) = a_j/(1-a_i),
    the left-hand sides recomputed by the oracle on the reduced cache."""
    rng = np.random.default_rng(100 + seed)
    n, d = 24, 16
    q, K, V = _rand_unit(rng, 1, d, n, qs=2.0)
    r = oracle.unit_attend(q, K, V)
    o, a, Vf = r["out"][0], r["alpha"][0], _f64(V)
    Vmax = np.linalg.norm(Vf, axis=1).max()
    for i in range(n):
        keep = [j for j in range(n) if j != i]
        ri = oracle.unit_attend(q, K[keep], V[keep])
        delta = o - ri["out"][0]
        c = a[i] * Vf[i]
        R = -a[i] / (1 - a[i]) * (o - c)
        np.testing.assert_allclose(delta, c + R, rtol=0, atol=1e-12)
        assert np.linalg.norm(delta - c) <= 2 * Vmax * a[i] / (1 - a[i]) + 1e-12
        np.testing.assert_allclose(ri["alpha"][0], a[keep] / (1 - a[i]), rtol=1e-12)


def test_query_drift_bound():
    """Eq. 12 / App. A: |alpha_{t+1}^i - alpha_t^i| <= max_j |Delta s_j|
    <= ||q_{t+1} - q_t|| max_j ||k_j|| / sqrt(d) (Cauchy-Schwarz form, the bf16 queries are
    not exactly unit-norm), on the synthetic query random walk."""
    wl = CONFIGS["tiny"]
    syn = Synth(wl, seed=3)
    K, V = syn.prefill(100)
    Kb, Vb = bits(K[0, 0]), bits(V[0, 0])
    q_prev = bits(syn.step()[0][0])
    for _ in range(20):
        q = bits(syn.step()[0][0])
        r0 = oracle.unit_attend(q_prev, Kb, Vb)
        r1 = oracle.unit_attend(q, Kb, Vb)
        dq = np.linalg.norm(_f64(q) - _f64(q_prev))
        kmax = np.linalg.norm(_f64(Kb), axis=1).max()
        bound = dq * kmax / math.sqrt(wl.d)
        assert np.abs(r1["alpha"] - r0["alpha"]).max() <= bound + 1e-12
        a, b = _f64(q).ravel(), _f64(q_prev).ravel()
        cos = float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b)))
        assert cos > 0.99          # the walk mirrors P:105 / P:626
        q_prev = q


# --- step protocol -------------------------------------------------------------------

def test_protocol_tiny_run():
    """C.3 #14: fill appends at slot n, then exactly one slot changes per
    step and the valid count stays N.  tiny config: prefill 16, N 128, 512 steps ->
    112 appends + 400 evictions."""
    wl = CONFIGS["tiny"]
    syn = Synth(wl, seed=0)
    c = oracle.OracleCache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N)
    K, V = syn.prefill()
    c.prefill(0, bits(K[0]), bits(V[0]))
    appends = evictions = 0
    for t in range(wl.steps):
        q, kn, vn = (bits(x) for x in syn.step())
        n_before = int(c.n_valid[0, 0])
        K0, V0 = c.K.copy(), c.V.copy()
        out, slot, scores = c.step(q, kn, vn)
        changed = np.nonzero(np.any(K0[0, 0] != c.K[0, 0], axis=1) | np.any(V0[0, 0] != c.V[0, 0], axis=1))[0]
        assert set(changed.tolist()) <= {int(slot[0, 0])}
        if n_before < wl.N:
            assert slot[0, 0] == n_before and c.n_valid[0, 0] == n_before + 1
            appends += 1
        else:
            assert c.n_valid[0, 0] == wl.N
            assert slot[0, 0] == int(np.argmin(scores[0, 0]))
            evictions += 1
        assert np.all(np.isinf(scores[0, 0, n_before:]))
        np.testing.assert_array_equal(c.K[0, 0, slot[0, 0]], kn[0, 0])
    assert (appends, evictions) == (112, 400)
    assert (wl.steps - (wl.N - wl.prefill)) == evictions


def test_threaded_step_equals_single_thread():
    wl = CONFIGS["tiny"]
    rng = np.random.default_rng(9)
    B, Hq, Hkv, d, N = 3, 8, 2, 32, 40
    caches = [oracle.OracleCache(B, Hq, Hkv, d, N, nthreads=t) for t in (1, 4)]
    K = _b(rng.standard_normal((B, Hkv, 30, d)))
    V = _b(rng.standard_normal((B, Hkv, 30, d)))
    for c in caches:
        for b in range(B):
            c.prefill(b, K[b], V[b])
    for _ in range(15):
        q = _b(rng.standard_normal((B, Hq, d)))
        kn, vn = _b(rng.standard_normal((B, Hkv, d))), _b(rng.standard_normal((B, Hkv, d)))
        r = [c.step(q, kn, vn) for c in caches]
        np.testing.assert_array_equal(r[0][0], r[1][0])
        np.testing.assert_array_equal(r[0][1], r[1][1])
    np.testing.assert_array_equal(caches[0].K, caches[1].K)


def test_deferred_mode_identity_with_same_step():
    """C.3 #16: deferred mode (Fig. 2 literal) with the newest token excluded from the
    candidates at budget N evicts the same TOKENS and yields the same outputs as same-step
    mode at budget N-1."""
    rng = np.random.default_rng(11)
    B, Hq, Hkv, d, N, P = 2, 4, 2, 16, 12, 5
    same = oracle.OracleCache(B, Hq, Hkv, d, N - 1)
    defer = oracle.OracleCache(B, Hq, Hkv, d, N)
    K = _b(rng.standard_normal((B, Hkv, P, d)))
    V = _b(rng.standard_normal((B, Hkv, P, d)))
    ids_same = np.full((B, Hkv, N - 1), -1)
    ids_def = np.full((B, Hkv, N), -1)
    for b in range(B):
        same.prefill(b, K[b], V[b])
        defer.prefill(b, K[b], V[b])
        ids_same[b, :, :P] = np.arange(P)
        ids_def[b, :, :P] = np.arange(P)
    for t in range(40):
        tok = P + t
        q = _b(rng.standard_normal((B, Hq, d)) * 2)
        kn, vn = _b(rng.standard_normal((B, Hkv, d))), _b(rng.standard_normal((B, Hkv, d)))
        o1, s1, _ = same.step(q, kn, vn)
        o2, written, pend, _ = defer.step_deferred(q, kn, vn, exclude_newest=True)
        np.testing.assert_allclose(o1, o2, rtol=1e-11, atol=1e-13)
        for b in range(B):
            for h in range(Hkv):
                ids_same[b, h, s1[b, h]] = tok
                ids_def[b, h, written[b, h]] = tok
                # the token the deferred run will overwrite next is the one same-step just evicted,
                # i.e. the two caches hold the same token sets once the newest is set aside
                live_def = set(ids_def[b, h].tolist()) - {-1}
                if defer.n_valid[b, h] == N:
                    live_def.discard(int(ids_def[b, h, pend[b, h]]))
                assert live_def == set(ids_same[b, h].tolist()) - {-1}
