"""Single-CTA streaming rate: U units of one kv head (G=4, d=128, budget N) with split_tokens=N (one CTA per
unit, S=1), so U CTAs stream N*512 B each.  Prints GB/s per CTA and total.
usage: python tools/percta_probe.py [N] [U list]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import timed_steps
from paper_2603_11504_b200 import Cache

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
Us = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,8,32,74,148").split(",")]
G, d = 4, 128
for U in Us:
    c = Cache(U, G, 1, d, N, out_dtype="bf16", split_tokens=N)
    K, V, nv = c.views()
    K.normal_(); V.normal_(); nv.fill_(N)
    q = torch.randn(U, G, d, device="cuda").bfloat16()
    kn = torch.randn(U, 1, d, device="cuda").bfloat16()
    vn = torch.randn(U, 1, d, device="cuda").bfloat16()
    out, slot, _ = c.new_outputs()
    st = torch.cuda.Stream()
    for _ in range(3):
        c.decode_step(q, kn, vn, out, slot, stream=st)
    torch.cuda.synchronize()

    def run(i):
        with torch.cuda.stream(st):
            for _ in range(10):
                c.decode_step(q, kn, vn, out, slot, stream=st)

    us = timed_steps(run, 10, st, None) * 1e3
    per = N * 512 / (us * 1e-6) / 1e9
    print(f"N={N} U={U} plan={c.plan()} {us:.1f} us/step  {per:.1f} GB/s per CTA  {per * U:.0f} GB/s total", flush=True)
    c.close()
    del c, K, V, nv
    torch.cuda.empty_cache()
