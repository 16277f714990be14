"""Plan exploration for one budget-sweep point: every split S (split_tokens = N / S rounded to a tile)
x k CTAs per SM x solo rounds, timed like tools/sweep.py (L2-cold caches), next to the automatic plan.
usage: python tools/split_explore.py --points 32x4096,32x8192 [--splits 1,2,3,4,5,6,7,8] [--out f.jsonl]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import alg_bytes_per_step, cache_bytes_per_gpu, layers_for, peaks, timed_steps
from lf_synth import Synth, random_cache, sweep_workload
from paper_2603_11504_b200 import Cache, LFError

ap = argparse.ArgumentParser()
ap.add_argument("--points", default="32x4096,32x8192")
ap.add_argument("--splits", default="0,1,2,3,4,5,6,7,8,12,16")
ap.add_argument("--ks", default="1,2")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--lat", default="auto", choices=["auto", "both"],
                help="both: time split plans with and without the latency variant")
ap.add_argument("--no-solo", action="store_true", help="skip the solo-round variants")
ap.add_argument("--out", default="gpurun_out/split_explore.jsonl")
args = ap.parse_args()
peak, _ = peaks()
f = open(args.out, "a")


def measure(B, N, **kw):
    wl = sweep_workload(B, N)
    cache = Cache(B, wl.Hq, wl.Hkv, wl.d, N, out_dtype="bf16", **kw)
    K, V, nv = cache.views()
    k0, v0 = random_cache(B, wl.Hkv, N, wl.d, device="cuda")
    K.copy_(k0); V.copy_(v0); nv.fill_(N)
    del k0, v0
    L = max(layers_for(cache_bytes_per_gpu(wl, B)), 1)
    layers = [cache]
    for _ in range(1, L):
        c2 = Cache(B, wl.Hq, wl.Hkv, wl.d, N, out_dtype="bf16", **kw)
        K2, V2, nv2 = c2.views()
        K2.copy_(K); V2.copy_(V); nv2.copy_(nv)
        layers.append(c2)
    syn = Synth(wl, device="cuda")
    pool = [syn.step() for _ in range(4)]
    out, slot, _ = cache.new_outputs()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    steps = max(3, min(args.steps, 2000 // L))
    for i in range(3):
        for c in layers:
            c.decode_step(*pool[i % 4], out, slot, stream=st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(steps):
            for c in layers:
                c.decode_step(*pool[i % 4], out, slot, stream=st)
    g.replay()
    torch.cuda.synchronize()

    def run(i):
        with torch.cuda.stream(st):
            g.replay()
    us = timed_steps(run, steps * L, st, None) * 1e3
    alg = alg_bytes_per_step(wl, B, 2)
    rec = {"B": B, "N": N, "kw": kw, "latency_us": us, "frac": alg / (us * 1e-6) / 1e9 / peak, "plan": cache.plan()}
    for c in layers:
        c.close()
    del layers, cache, g
    torch.cuda.empty_cache()
    return rec


for pt in args.points.split(","):
    B, N = map(int, pt.split("x"))
    for S in map(int, args.splits.split(",")):
        split = 0 if S == 0 else ((N + S - 1) // S + 127) // 128 * 128
        if S and -(-N // split) != S:
            continue
        for k in (map(int, args.ks.split(",")) if S else [0]):
            for solo in ((None,) if S in (0, 1) or args.no_solo else (False, True)):
                for lat in ((None,) if S in (0, 1) or args.lat == "auto" else (False, True)):
                    kw = dict(split_tokens=split, ctas_per_sm=k, solo=solo, latency_variant=lat)
                    try:
                        rec = measure(B, N, **kw)
                    except LFError as e:
                        print("no plan", B, N, kw, str(e)[:120], flush=True)
                        continue
                    print(json.dumps(rec), flush=True)
                    f.write(json.dumps(rec) + "\n")
                    f.flush()
