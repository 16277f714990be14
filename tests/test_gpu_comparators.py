"""NEXT-f2 comparators against the oracle (Fig. 1, P:333 the throughput gap to FullKV):

  * FullKV = the same fused kernel in append mode with a budget that holds the whole generation
    (prefill + every decode token): the cache grows n -> T, no token is ever evicted, and every
    step's output is full attention over all tokens so far;
  * the unfused library pipeline of tools/compare.py (torch/cuBLAS: logits, softmax, PV, a separate
    score pass over V, argmin, scatter) -- the Fig. 1 shape of the comparison.

Both are timed by tools/compare.py (context only); here they must compute what the oracle computes.
"""
import os
import sys

import numpy as np
import pytest
import torch

import oracle
from lf_synth import Synth, Workload, bits
from tests.parity import Stats, accept_slots, check_out, run_lockstep, setup_pair

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("G,d,prefill,steps", [(4, 128, 100, 300), (7, 128, 37, 200), (1, 64, 10, 150)])
def test_fullkv_append_mode_grows_to_T(cuda_lib, G, d, prefill, steps):
    """Budget T = prefill + steps: every step appends (slot = n, n -> n+1), nothing is evicted, and
    out / scores / cache match the oracle step by step until the cache holds all T tokens."""
    T = prefill + steps
    wl = Workload("fullkv", 2, 2 * G, 2, d, T, prefill, steps)
    cache, orc, syn = setup_pair(wl, seed=T, nthreads=4)
    st = run_lockstep(cache, orc, syn, steps)
    assert st.evictions == 0
    assert (cache.views()[2].cpu().numpy() == T).all()


def test_unfused_pipeline_matches_oracle(cuda_lib):
    """tools/compare.py's unfused library pipeline, stepped on the oracle's inputs: fp32 out within
    the 2e-3 bar, the oracle's victim (up to accepted near-ties), and the same cache afterwards."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from compare import unfused_step
    B, Hq, Hkv, d, N, steps = 3, 16, 4, 128, 640, 6
    wl = Workload("unfused", B, Hq, Hkv, d, N, N, steps)
    syn = Synth(wl, seed=21)
    orc = oracle.OracleCache(B, Hq, Hkv, d, N, nthreads=4)
    K0, V0 = syn.prefill()
    for b in range(B):
        orc.prefill(b, bits(K0[b]), bits(V0[b]))
    Kd, Vd = K0.cuda().contiguous(), V0.cuda().contiguous()
    st = Stats()
    for _ in range(steps):
        q, kn, vn = syn.step()
        out, slot = unfused_step(Kd, Vd, N, q.cuda(), kn.cuda(), vn.cuda(), d ** -0.5, Hq // Hkv)
        torch.cuda.synchronize()
        nv = orc.n_valid.copy()
        o_ref, s_ref, sc_ref = orc.compute(bits(q), bits(kn), bits(vn))
        check_out(out.double().cpu().numpy(), o_ref, "f32", st)
        sl = slot.int().cpu().numpy()
        chosen = accept_slots(sl, s_ref, sc_ref, nv, N, st)
        assert (chosen == sl).all(), "the unfused pipeline's slot is not an accepted victim"
        orc.apply(bits(kn), bits(vn), chosen)
    np.testing.assert_array_equal(bits(Kd.cpu()), orc.K)
    np.testing.assert_array_equal(bits(Vd.cpu()), orc.V)
    assert st.max_out_err < 1e-5, st
