"""Debug: a few decode steps of one forced plan (for compute-sanitizer runs).
usage: python tools/dbg/one_step.py B Hq Hkv N split_tokens ctas_per_sm lat(0/1/2) [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from lf_synth import Synth, Workload
from paper_2603_11504_b200 import Cache
B, Hq, Hkv, N, split, k, lat = map(int, sys.argv[1:8])
steps = int(sys.argv[8]) if len(sys.argv) > 8 else 3
wl = Workload("dbg", B, Hq, Hkv, 128, N, N - 1, steps)
c = Cache(B, Hq, Hkv, 128, N, split_tokens=split, ctas_per_sm=k, latency_variant={0: None, 1: False, 2: True}[lat])
syn = Synth(wl, seed=1)
K, V = syn.prefill()
for b in range(B):
    c.prefill(b, K[b].cuda(), V[b].cuda())
out, slot, sc = c.new_outputs(with_scores=True)
for _ in range(steps):
    q, kn, vn = syn.step()
    c.decode_step(q.cuda(), kn.cuda(), vn.cuda(), out, slot, sc)
torch.cuda.synchronize()
print("ok", c.plan())
