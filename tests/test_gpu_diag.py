"""GPU diagnostics kernel (NEXT-f4) against the oracle: LongFlow victim, exact-objective victim (Eq. 3's
right-hand side, which the kernel evaluates with App. A's exact remainder P:424-426 and the oracle by
brute-force re-attention without each token), remainder bound."""
import numpy as np
import pytest
import torch

import oracle
from lf_synth import Synth, Workload, bits

pytestmark = pytest.mark.gpu


def _near(vals, i, j, rtol=1e-4):
    return vals[i] <= (1 + rtol) * vals[j] + 1e-30


@pytest.mark.parametrize("G,d,N,pre", [(4, 128, 300, 300), (1, 64, 128, 128), (7, 128, 513, 400)])
def test_diag_matches_oracle(cuda_lib, G, d, N, pre):
    from paper_2603_11504_b200 import Cache
    B, Hkv = 2, 2
    wl = Workload("diag", B, G * Hkv, Hkv, d, N, pre, 3)
    syn = Synth(wl, seed=G)
    cache = Cache(B, G * Hkv, Hkv, d, N)
    K, V = syn.prefill()
    for b in range(B):
        cache.prefill(b, K[b].cuda(), V[b].cuda())
    q, kn, vn = syn.step()
    islot, fstat = cache.diagnose_step(q.cuda(), kn.cuda(), vn.cuda())
    torch.cuda.synchronize()
    islot, fstat = islot.cpu().numpy(), fstat.cpu().numpy()
    for b in range(B):
        for h in range(Hkv):
            r = oracle.unit_attend(bits(q[b, h * G:(h + 1) * G]), bits(K[b, h]), bits(V[b, h]), bits(kn[b, h]),
                                   bits(vn[b, h]))
            # the exact objective by brute force: the unit re-attended without each token (oracle/)
            E = oracle.exact_objective(bits(q[b, h * G:(h + 1) * G]), bits(K[b, h]), bits(V[b, h]),
                                       bits(kn[b, h]), bits(vn[b, h]))
            lf, ex, rank = islot[b, h]
            assert lf == r["slot"] or _near(r["scores"], lf, r["slot"])
            assert ex == int(np.argmin(E)) or _near(E, ex, int(np.argmin(E)))
            np.testing.assert_allclose(fstat[b, h, 0], E[lf], rtol=1e-3)
            np.testing.assert_allclose(fstat[b, h, 1], E[ex], rtol=1e-3)
            assert abs(rank - int((E < E[lf]).sum())) <= 2
            assert 0 < fstat[b, h, 2] <= 1.0 + 1e-6   # remainder within the App. A bound
