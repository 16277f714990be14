"""Is the `r` step slower under the sustained power cap because of its own SM work, or because the
whole memory path slows with the capped clock?  Times, back to back in one process and each for ~2 s
(long enough for sw_power_cap to engage), with the SM clock sampled during each: (1) the `r` decode
step (CUDA graph of 200 steps, 8.6 GB per step), (2) a read-only stream of the same 8.6 GB (torch
sum over the cache, the kernel's access pattern minus all compute), (3) a device copy of 4.3 GB
(read + write 8.6 GB, MEASURED_PEAKS' method).  Prints GB/s and median SM MHz for each.
usage: python tools/sustained_probe.py [--seconds 2]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import ClockSampler, alg_bytes_per_step
from lf_synth import CONFIGS, Synth, random_cache
from paper_2603_11504_b200 import Cache

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=2.0)
ap.add_argument("--rounds", type=int, default=2)
args = ap.parse_args()
wl = CONFIGS["r"]
cache = Cache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N, out_dtype="bf16")
K, V, nv = cache.views()
k0, v0 = random_cache(wl.B, wl.Hkv, wl.N, wl.d, device="cuda")
K.copy_(k0)
V.copy_(v0)
nv.fill_(wl.N)
del k0, v0
syn = Synth(wl, device="cuda")
pool = [syn.step() for _ in range(4)]
out, slot, _ = cache.new_outputs()
torch.cuda.synchronize()
st = torch.cuda.Stream()
nb = cache._buf.numel() // 16 * 16
kv = cache._buf[:nb].view(torch.float32)   # the whole slab (K + V): the read-only stream's input
half = kv.numel() // 2
dst = torch.empty(half, dtype=torch.float32, device="cuda")
sink = torch.empty((), dtype=torch.float32, device="cuda")


def graph_of(fn, n):
    with torch.cuda.stream(st):
        for i in range(3):
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(n):
            fn(i)
    return g


def timed(g, n, nbytes):
    reps = 0
    ms_tot = 0.0
    with ClockSampler(0) as clk:
        t0 = time.time()
        while time.time() - t0 < args.seconds:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            with torch.cuda.stream(st):
                g.replay()
            e1.record(st)
            e1.synchronize()
            ms_tot += e0.elapsed_time(e1)
            reps += 1
    per = ms_tot / (reps * n)
    return {"ms_per_op": per, "GBps": nbytes / (per * 1e-3) / 1e9, "clocks": clk.summary()}


steps = 200
g_r = graph_of(lambda i: cache.decode_step(*pool[i % 4], out, slot, stream=st), steps)
g_read = graph_of(lambda i: torch.sum(kv[: 2 * half], dim=0, out=sink), 20)
g_copy = graph_of(lambda i: dst.copy_(kv[:half]), 20)
alg = alg_bytes_per_step(wl, wl.B, 2)
res = []
for r in range(args.rounds):
    for name, g, n, nbytes in (("r decode step", g_r, steps, alg), ("read-only stream (sum)", g_read, 20, 8 * half),
                               ("device copy", g_copy, 20, 8 * half)):
        d = timed(g, n, nbytes)
        d["what"] = name
        d["round"] = r
        print(json.dumps(d), flush=True)
        res.append(d)
