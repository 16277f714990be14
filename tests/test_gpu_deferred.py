"""GPU parity of the Fig. 2-literal deferred eviction mode (NEXT-f1) against the oracle's
lfo_step_deferred, for both kernels, with and without the newest token as a candidate."""
import numpy as np
import pytest
import torch

import oracle
from lf_synth import Synth, Workload, bits
from tests.parity import SCORE_ATOL, SCORE_RTOL, Stats, check_out, check_scores
from tests.test_gpu_parity import _need

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["deferred", "deferred_exclude_newest"])
@pytest.mark.parametrize("kernel,G,d", [("simt", 1, 64), ("simt", 4, 128), ("tcgen05", 4, 128),
                                        ("tcgen05", 7, 128)])
def test_deferred_lockstep(cuda_lib, mode, kernel, G, d):
    _need(kernel, G, d)
    from paper_2603_11504_b200 import Cache
    B, Hkv, N, pre, steps = 3, 2, 300, 290, 30
    wl = Workload("defer", B, G * Hkv, Hkv, d, N, pre, steps)
    syn = Synth(wl, seed=G + d)
    cache = Cache(B, wl.Hq, Hkv, d, N, kernel=kernel, mode=mode, split_tokens=128)
    orc = oracle.OracleCache(B, wl.Hq, Hkv, d, N)
    K, V = syn.prefill()
    for b in range(B):
        cache.prefill(b, K[b].cuda(), V[b].cuda())
        orc.prefill(b, bits(K[b]), bits(V[b]))
    out, slot, scores = cache.new_outputs(with_scores=True)
    st = Stats()
    excl = mode.endswith("newest")
    for t in range(steps):
        q, kn, vn = syn.step()
        cache.decode_step(q.cuda(), kn.cuda(), vn.cuda(), out, slot, scores)
        torch.cuda.synchronize()
        o_ref, written, pend_ref, sc_ref = orc.step_deferred(bits(q), bits(kn), bits(vn), exclude_newest=excl)
        np.testing.assert_array_equal(slot.cpu().numpy(), written)
        check_out(out.cpu().double().numpy(), o_ref, "f32", st)
        check_scores(scores.cpu().numpy(), sc_ref, orc.n_valid, st)
        pend = cache.pending().cpu().numpy()
        for u in np.ndindex(pend.shape):
            if pend[u] != pend_ref[u]:
                cand = [j for j in range(orc.n_valid[u]) if not (excl and j == written[u])]
                m = min(sc_ref[u][j] for j in cand)
                assert sc_ref[u][pend[u]] <= (1 + SCORE_RTOL) * m + SCORE_ATOL, (u, pend[u], pend_ref[u])
                orc.pend[u] = pend[u]
                st.adoptions += 1
    Kc, Vc, nv = cache.views()
    np.testing.assert_array_equal(bits(Kc), orc.K)
    np.testing.assert_array_equal(nv.cpu().numpy(), orc.n_valid)
    print(mode, kernel, G, st)


def test_deferred_cross_mode_identity_on_gpu(cuda_lib):
    """C.3 #16 on the CUDA path: deferred (newest excluded) at N == same-step at N-1, token by token."""
    from paper_2603_11504_b200 import Cache
    B, G, Hkv, d, N, pre = 2, 4, 2, 128, 260, 250
    wl = Workload("x", B, G * Hkv, Hkv, d, N, pre, 40)
    a = Cache(B, G * Hkv, Hkv, d, N - 1, kernel="tcgen05", split_tokens=128)
    b = Cache(B, G * Hkv, Hkv, d, N, kernel="tcgen05", split_tokens=128, mode="deferred_exclude_newest")
    syn = Synth(wl, seed=3)
    K, V = syn.prefill()
    for s in range(B):
        a.prefill(s, K[s].cuda(), V[s].cuda())
        b.prefill(s, K[s].cuda(), V[s].cuda())
    oa, sa, _ = a.new_outputs()
    ob, sb, _ = b.new_outputs()
    for t in range(40):
        q, kn, vn = (x.cuda() for x in syn.step())
        a.decode_step(q, kn, vn, oa, sa)
        b.decode_step(q, kn, vn, ob, sb)
        torch.cuda.synchronize()
        err = (oa - ob).abs().max() / oa.abs().max()
        assert float(err) < 1e-5
    # the same set of tokens survives (compare rows as sets, ignoring the pending victim of b)
    Ka, _, _ = a.views()
    Kb, _, _ = b.views()
    pend = b.pending().cpu().numpy()
    for s in range(B):
        for h in range(Hkv):
            ra = {bytes(r) for r in bits(Ka[s, h]).view(np.uint8).reshape(N - 1, -1)}
            rb = [bytes(r) for r in bits(Kb[s, h]).view(np.uint8).reshape(N, -1)]
            del rb[pend[s, h]]
            assert ra == set(rb)


@pytest.mark.parametrize("mode", ["deferred", "deferred_exclude_newest"])
def test_deferred_full_prefill_is_a_protocol_error(cuda_lib, mode):
    """R26: in the Fig. 2-literal modes a step's token covers the slot chosen at the PREVIOUS step
    (P:152).  A sequence prefilled to the whole budget has none, so lf_decode_step refuses it
    (LF_ERR_INVALID_ARGUMENT, before any launch) -- as the oracle's lfo_step_deferred does -- and a
    re-prefill below the budget clears the state (and the stale pending victim of the sequence)."""
    from paper_2603_11504_b200 import Cache, LFError
    B, Hq, Hkv, d, N = 2, 8, 2, 128, 64
    wl = Workload("defer_full", B, Hq, Hkv, d, N, N, 1)
    syn = Synth(wl, seed=3)
    cache = Cache(B, Hq, Hkv, d, N, mode=mode)
    orc = oracle.OracleCache(B, Hq, Hkv, d, N)
    K, V = syn.prefill()
    cache.prefill(0, K[0, :, :N - 4].cuda(), V[0, :, :N - 4].cuda())
    cache.prefill(1, K[1].cuda(), V[1].cuda())                       # full: no victim chosen yet
    orc.prefill(0, bits(K[0, :, :N - 4]), bits(V[0, :, :N - 4]))
    orc.prefill(1, bits(K[1]), bits(V[1]))
    q, kn, vn = syn.step()
    out, slot, _ = cache.new_outputs()
    with pytest.raises(LFError) as e:
        cache.decode_step(q.cuda(), kn.cuda(), vn.cuda(), out, slot)
    assert e.value.status == 1 and "sequence 1" in str(e.value)
    with pytest.raises(oracle.OracleError):
        orc.step_deferred(bits(q), bits(kn), bits(vn), exclude_newest=mode.endswith("newest"))
    # the pending victims were reset by the prefill
    assert (cache.pending().cpu().numpy() == -1).all()
    cache.prefill(1, K[1, :, :N - 1].cuda(), V[1, :, :N - 1].cuda())   # below the budget: fine again
    cache.decode_step(q.cuda(), kn.cuda(), vn.cuda(), out, slot)
    torch.cuda.synchronize()
    assert slot.cpu().numpy().tolist() == [[N - 4] * Hkv, [N - 1] * Hkv]
