"""Pins for the oracle's SnapKV prefill selection (NEXT-f3)."""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from lf_synth import bits, bf16

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _b(x):
    return bits(bf16(x))


def test_hand_example():
    g = json.load(open(os.path.join(GOLD, "snapkv_example.json")))
    r1 = oracle.snapkv_select(_b(g["q_obs"]), _b(g["K"]), g["budget"], pool_kernel=1, scale=math.log(2))
    np.testing.assert_allclose(r1["score"], g["score"], atol=1e-15)
    np.testing.assert_array_equal(r1["kept"], g["kept_ks1"])
    r3 = oracle.snapkv_select(_b(g["q_obs"]), _b(g["K"]), g["budget"], pool_kernel=3, scale=math.log(2))
    np.testing.assert_allclose(r3["pooled"], g["pooled_ks3"], atol=1e-15)
    np.testing.assert_array_equal(r3["kept"], g["kept_ks3"])


def _torch_route(q_obs, K, budget, ks, scale):
    """Independent library route: causal attention of the window queries (torch softmax with a
    mask), mean over (head, query), F.max_pool1d 'same', torch.topk, sort."""
    q = torch.from_numpy(oracle.bf16_bits_to_f64(q_obs))          # [G][w][d]
    Kf = torch.from_numpy(oracle.bf16_bits_to_f64(K))             # [n][d]
    G, w, d = q.shape
    n = Kf.shape[0]
    s = torch.einsum("gwd,nd->gwn", q, Kf) * scale
    pos = torch.arange(n)
    qpos = n - w + torch.arange(w)
    s = s.masked_fill(pos[None, None, :] > qpos[None, :, None], float("-inf"))
    a = torch.softmax(s, dim=-1)
    score = a[..., : n - w].mean(dim=(0, 1))
    pooled = torch.nn.functional.max_pool1d(score[None, None], ks, stride=1, padding=(ks - 1) // 2)[0, 0]
    # pooling creates exact ties: the rule is "larger pooled first, then lower index" (R24), i.e. a
    # stable descending sort
    top = torch.sort(-pooled, stable=True).indices[: budget - w].sort().values
    return np.concatenate([top.numpy(), np.arange(n - w, n)]), score.numpy(), pooled.numpy()


@pytest.mark.parametrize("G,w,n,budget,ks", [(1, 4, 40, 20, 7), (4, 8, 200, 64, 7), (2, 32, 300, 128, 5),
                                            (7, 3, 90, 10, 1)])
def test_matches_torch_route(G, w, n, budget, ks):
    rng = np.random.default_rng(n + G)
    d = 16
    q = _b(rng.standard_normal((G, w, d)) * 2)
    K = _b(rng.standard_normal((n, d)))
    r = oracle.snapkv_select(q, K, budget, pool_kernel=ks)
    kept, score, pooled = _torch_route(q, K, budget, ks, 1 / math.sqrt(d))
    np.testing.assert_allclose(r["score"], score, rtol=1e-12)
    np.testing.assert_allclose(r["pooled"], pooled, rtol=1e-12)
    np.testing.assert_array_equal(r["kept"], kept)
    # invariants: |kept| == budget, the window kept, ascending, unique
    assert len(r["kept"]) == budget
    assert list(r["kept"][-w:]) == list(range(n - w, n))
    assert np.all(np.diff(r["kept"]) > 0)


def test_near_zero_token_dropped():
    """n = budget + 1 with one token of near-zero weight -> that token is dropped."""
    rng = np.random.default_rng(0)
    d, n, w = 8, 6, 2
    q = _b(np.ones((1, w, d)))
    K = _b(rng.uniform(-0.2, 0.2, (n, d)))
    K[2] = _b(np.full(d, -6.0))
    r = oracle.snapkv_select(q, K, n - 1, pool_kernel=1)
    assert 2 not in r["kept"] and len(r["kept"]) == n - 1


def test_rejects_no_compression_needed():
    with pytest.raises(oracle.OracleError):
        oracle.snapkv_select(_b(np.ones((1, 1, 4))), _b(np.ones((4, 4))), 4)
