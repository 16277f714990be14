"""NEXT-f4: the paper's approximations checked at B200 scale on a synthetic long-output trajectory.
Before each decode step the diagnostics kernel compares LongFlow's victim (Eq. 6) with the victim of
the exact eviction objective for the current query (Eq. 3 RHS, exact via App. A); reported: agreement
rate, mean rank of LongFlow's victim under the exact objective (as a fraction of the cache), the
mean E ratio, the max remainder-bound ratio (must be <= 1), and the query drift bound Eq. 12
 in its Cauchy-Schwarz form, max |Delta s| <= ||q_{t+1} - q_t|| max ||k|| / sqrt(d).
usage: python tools/diag_run.py [--workload q3] [--steps 16]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import workload_of
from lf_synth import Synth
from paper_2603_11504_b200 import Cache

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="q3")
ap.add_argument("--steps", type=int, default=16)
ap.add_argument("--out", default="gpurun_out/diag.json")
args = ap.parse_args()
wl = workload_of(args.workload)
syn = Synth(wl, device="cuda")
cache = Cache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N, out_dtype="bf16")
K, V, nv = cache.views()
K.normal_()
V.normal_()
nv.fill_(wl.N)
out, slot, _ = cache.new_outputs()
agree, rank, eratio, rmax, drift_ok = [], [], [], 0.0, True
q_prev = None
kmax = float(K.float().norm(dim=-1).max())
for t in range(args.steps):
    q, kn, vn = syn.step()
    islot, fstat = cache.diagnose_step(q, kn, vn)
    cache.decode_step(q, kn, vn, out, slot)
    torch.cuda.synchronize()
    agree.append(float((islot[..., 0] == islot[..., 1]).float().mean()))
    rank.append(float((islot[..., 2].float() / wl.N).mean()))
    eratio.append(float((fstat[..., 0] / fstat[..., 1].clamp_min(1e-30)).mean()))
    rmax = max(rmax, float(fstat[..., 2].max()))
    if q_prev is not None:   # Eq. 12 bound on the logit drift between adjacent queries (per q head)
        dq = (q.float() - q_prev.float()).norm(dim=-1)                        # [B][Hq]
        bound = dq * kmax / wl.d ** 0.5
        G = wl.G
        ds = torch.einsum("bhd,bhnd->bhn", (q.float() - q_prev.float()).view(wl.B * wl.Hkv, G, wl.d),
                          K.float().view(wl.B * wl.Hkv, 1, wl.N, wl.d).expand(-1, G, -1, -1)).abs().amax(-1)
        drift_ok &= bool((ds / wl.d ** 0.5 <= bound.view(wl.B * wl.Hkv, G) * (1 + 1e-5) + 1e-6).all())
    q_prev = q
res = {"workload": wl.tag, "steps": args.steps, "units": wl.B * wl.Hkv,
       "agreement_rate": sum(agree) / len(agree), "mean_rank_fraction": sum(rank) / len(rank),
       "mean_E_ratio_longflow_over_exact": sum(eratio) / len(eratio), "max_remainder_bound_ratio": rmax,
       "eq12_drift_bound_holds": drift_ok}
print(json.dumps(res))
open(args.out, "w").write(json.dumps(res) + "\n")
