"""Roofline fraction across GQA group sizes and head dims at a bandwidth-bound size (B x Hkv=8, N).
usage: python tools/gsweep.py [--out gpurun_out/gsweep.jsonl]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import alg_bytes_per_step, peaks
from lf_synth import Synth, Workload, random_cache
from paper_2603_11504_b200 import Cache

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/gsweep.jsonl")
ap.add_argument("--only-g", type=int, default=0, help="restrict to one group size")
args = ap.parse_args()
peak, _ = peaks()
f = open(args.out, "w")
for (G, d, kernel) in [(1, 128, "auto"), (1, 128, "simt"), (1, 64, "simt"), (2, 128, "auto"), (2, 128, "simt"),
                       (4, 128, "auto"), (4, 128, "simt"), (7, 128, "auto"), (8, 128, "auto"), (8, 64, "simt")]:
    if args.only_g and G != args.only_g:
        continue
    B, Hkv, N = 256, 8, 4096
    wl = Workload(f"g{G}_d{d}", B, G * Hkv, Hkv, d, N, 0, 0)
    cache = Cache(B, wl.Hq, Hkv, d, N, out_dtype="bf16", kernel=kernel)
    K, V, nv = cache.views()
    k0, v0 = random_cache(B, Hkv, N, d, device="cuda")
    K.copy_(k0); V.copy_(v0); nv.fill_(N)
    del k0, v0
    syn = Synth(wl, device="cuda")
    pool = [syn.step() for _ in range(4)]
    out, slot, _ = cache.new_outputs()
    st = torch.cuda.Stream()
    for i in range(4):
        cache.decode_step(*pool[i % 4], out, slot, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(20):
            cache.decode_step(*pool[i % 4], out, slot, stream=st)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    alg = alg_bytes_per_step(wl, B, 2)
    rec = {"G": G, "d": d, "kernel": cache.plan()["kernel"], "B": B, "N": N, "latency_us": us,
           "frac_measured_peak": alg / (us * 1e-6) / 1e9 / peak}
    print(json.dumps(rec), flush=True)
    f.write(json.dumps(rec) + "\n")
    cache.close()
    del cache, K, V, nv, g
    torch.cuda.empty_cache()
