"""BASELINE configs[4]: budget sweep 512-16384 x batch 1-512 at fixed 80 % compression (32/8 GQA, d=128):
latency and HBM GB/s per point (full cache, every step evicts), one JSON line per point.
usage: python tools/sweep.py [--out gpurun_out/sweep.jsonl] [--steps 20] [--per-row 300]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import alg_bytes_per_step, cache_bytes_per_gpu, l2_note, layers_for, peaks, timed_steps
from lf_synth import Synth, random_cache, sweep_workload
from paper_2603_11504_b200 import Cache

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/sweep.jsonl")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--budgets", default="512,1024,2048,4096,8192,16384")
ap.add_argument("--batches", default="1,2,4,8,16,32,64,128,256,512")
ap.add_argument("--per-row", type=float, default=0.0,
                help="run each budget row in its own process with this timeout (s); a stalled row is "
                     "reported and skipped (DESIGN.md section 14)")
args = ap.parse_args()
if args.per_row > 0:
    import subprocess
    with open(args.out, "w") as f:
        for N in args.budgets.split(","):
            tmp = args.out + f".row{N}"
            cmd = [sys.executable, os.path.abspath(__file__), "--out", tmp, "--steps", str(args.steps),
                   "--budgets", N, "--batches", args.batches]
            try:
                subprocess.run(cmd, timeout=args.per_row, check=False)
            except subprocess.TimeoutExpired:
                print(f"row N={N}: timed out after {args.per_row:.0f} s", file=sys.stderr, flush=True)
            if os.path.exists(tmp):
                f.write(open(tmp).read())
                os.remove(tmp)
    sys.exit(0)
peak, _ = peaks()
f = open(args.out, "w")
for N in map(int, args.budgets.split(",")):
    for B in map(int, args.batches.split(",")):
        wl = sweep_workload(B, N)
        t0 = time.time()
        tl = {}
        cache = Cache(B, wl.Hq, wl.Hkv, wl.d, N, out_dtype="bf16")
        K, V, nv = cache.views()
        k0, v0 = random_cache(B, wl.Hkv, N, wl.d, device="cuda")
        K.copy_(k0); V.copy_(v0); nv.fill_(N)
        torch.cuda.synchronize()   # the decode steps below run on another stream
        del k0, v0
        syn = Synth(wl, device="cuda")
        pool = [syn.step() for _ in range(4)]
        out, slot, _ = cache.new_outputs()
        st = torch.cuda.Stream()
        for i in range(5):
            cache.decode_step(*pool[i % 4], out, slot, stream=st)
        torch.cuda.synchronize()
        tl["setup"] = time.time() - t0
        flush = g = None
        cb = cache_bytes_per_gpu(wl, B)
        L = layers_for(cb)
        layers = [cache]
        for _ in range(1, max(L, 1)):   # L2-resident cache: cycle L layer caches (bench.py, D.4)
            c2 = Cache(B, wl.Hq, wl.Hkv, wl.d, N, out_dtype="bf16")
            K2, V2, nv2 = c2.views()
            K2.copy_(K); V2.copy_(V); nv2.copy_(nv)
            layers.append(c2)
        torch.cuda.synchronize()   # copies on the default stream before the steps on `st`
        tl["layers"] = time.time() - t0
        steps = max(3, min(args.steps, 2000 // max(L, 1)))   # bounded graph size (<= ~2000 launches)
        if L == 0:
            flush = torch.zeros(128 << 20, dtype=torch.float32, device="cuda")
            run = lambda i: cache.decode_step(*pool[i % 4], out, slot, stream=st)
        else:
            for i in range(3):
                for c in layers:
                    c.decode_step(*pool[i % 4], out, slot, stream=st)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for i in range(steps):
                    for c in layers:
                        c.decode_step(*pool[i % 4], out, slot, stream=st)
            g.replay(); torch.cuda.synchronize()

            def run(i):
                with torch.cuda.stream(st):
                    g.replay()
        tl["graph"] = time.time() - t0
        us = timed_steps(run, steps * max(L, 1), st, flush) * 1e3
        tl["timed"] = time.time() - t0
        alg = alg_bytes_per_step(wl, B, 2)
        rec = {"B": B, "N": N, "latency_us": us, "tokens_per_s": B / (us * 1e-6), "alg_bytes": alg,
               "GBps": alg / (us * 1e-6) / 1e9, "frac_measured_peak": alg / (us * 1e-6) / 1e9 / peak,
               "plan": cache.plan(), "l2": l2_note(cb), "layer_caches": max(L, 1)}
        print(json.dumps(rec), flush=True)
        f.write(json.dumps(rec) + "\n")
        f.flush()
        for c in layers:
            c.close()
        del cache, K, V, nv, pool, out, slot, flush, g, layers
        torch.cuda.empty_cache()
        tl["closed"] = time.time() - t0
        print("phase times (s, cumulative):", {k: round(v, 2) for k, v in tl.items()}, file=sys.stderr, flush=True)
