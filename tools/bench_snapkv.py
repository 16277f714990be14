"""NEXT-f3 measurement: SnapKV prefill compression latency per sequence (all kv heads).
Work: 2 passes of R x n x d bf16 MACs (R = G * w observation rows) on the tensor cores (tcgen05) + the
K reads and the gather.  Rooflines reported: the measured dense bf16 tensor peak (MEASURED_PEAKS.json
bf16_tflops, burst) for the flops, and the HBM copy peak for the bytes (K read twice + kept K/V rows
read and written); at these sizes the step is latency-bound (6 launches, 2 of them one CTA per head).
usage: python tools/bench_snapkv.py [--out gpurun_out/snapkv_bench.jsonl]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11504_b200 import Cache

_pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
PEAK_BF16 = float(_pk["bf16_tflops"]) * 1e12
PEAK_HBM = float(_pk["hbm_gbs"]) * 1e9

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/snapkv_bench.jsonl")
args = ap.parse_args()
f = open(args.out, "w")
for (Hkv, G, n, N, w) in [(8, 4, 8192, 2048, 32), (8, 4, 32768, 3200, 32), (4, 7, 16384, 2048, 16)]:
    d = 128
    k = torch.randn(Hkv, n, d, device="cuda").to(torch.bfloat16)
    v = torch.randn(Hkv, n, d, device="cuda").to(torch.bfloat16)
    q = (2 * torch.randn(Hkv * G, w, d, device="cuda")).to(torch.bfloat16)
    cache = Cache(1, Hkv * G, Hkv, d, N, out_dtype="bf16")
    for _ in range(2):
        ws = cache.prefill_snapkv(0, k, v, q, window=w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        ws = cache.prefill_snapkv(0, k, v, q, window=w)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    flops = 2 * 2.0 * Hkv * G * w * n * d
    byts = 2 * Hkv * n * d * 2 + 2 * 2 * Hkv * N * d * 2
    rec = {"Hkv": Hkv, "G": G, "n": n, "budget": N, "window": w, "us": us, "TFLOPs": flops / (us * 1e-6) / 1e12,
           "frac_bf16_tensor_peak": flops / (us * 1e-6) / PEAK_BF16, "GBps": byts / (us * 1e-6) / 1e9,
           "frac_hbm_peak": byts / (us * 1e-6) / PEAK_HBM, "bound": "latency (tensor/hbm fractions both small)"}
    print(json.dumps(rec), flush=True)
    f.write(json.dumps(rec) + "\n")
    del cache, k, v, q, ws
