"""Debug: where do the 1-GPU and sharded runs (or two 1-GPU runs) differ?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from lf_synth import Workload
from tests.test_gpu_plans import _shard_run

for (tag, B, Hq, Hkv, N, P, od) in [("q3", 64, 32, 8, 4096, 2, "f32"), ("r", 256, 32, 8, 8192, 8, "f32")]:
    wl = Workload(tag, B, Hq, Hkv, 128, N, 0, 2)
    res, views, plans = _shard_run(wl, P, 2, seed=7, out_dtype=od)
    res2, _, _ = _shard_run(wl, P, 2, seed=7, out_dtype=od)
    for t in range(2):
        f, s = res[t]
        f2, s2 = res2[t]
        for i, nm in enumerate(("out", "slot", "scores")):
            d_fs = (f[i] != s[i])
            d_ff = (f[i] != f2[i])
            d_ss = (s[i] != s2[i])
            print(tag, "step", t, nm, "full!=shard", int(d_fs.sum()), "full!=full2", int(d_ff.sum()), "shard!=shard2", int(d_ss.sum()))
            if nm == "out" and d_fs.any():
                idx = d_fs.nonzero()
                units = sorted(set((int(b), int(h) // (Hq // Hkv)) for b, h, _ in idx.tolist()))
                print("   differing units (b, kvh):", units[:20], "of", len(units))
                rel = ((f[i] - s[i]).abs().max() / f[i].abs().max()).item()
                print("   max rel diff", rel)
