"""Where the small-config step latency goes: the same decode step timed (a) in a CUDA graph back to
back (PDL overlap), (b) one launch per event pair, warm L2, (c) one launch per event pair after a
512 MB L2 flush (what bench.py reports for L2-resident caches).
usage: python tools/latency_probe.py q7 [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import timed_steps, workload_of
from lf_synth import Synth, random_cache
from paper_2603_11504_b200 import Cache

w = sys.argv[1] if len(sys.argv) > 1 else "q7"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
wl = workload_of(w)
cache = Cache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N, out_dtype="bf16")
K, V, nv = cache.views()
k0, v0 = random_cache(wl.B, wl.Hkv, wl.N, wl.d, device="cuda")
K.copy_(k0); V.copy_(v0); nv.fill_(wl.N)
syn = Synth(wl, device="cuda")
pool = [syn.step() for _ in range(4)]
out, slot, _ = cache.new_outputs()
st = torch.cuda.Stream()
step = lambda i: cache.decode_step(*pool[i % 4], out, slot, stream=st)
for i in range(5):
    step(i)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for i in range(steps):
        step(i)
g.replay(); torch.cuda.synchronize()


def graph_run(i):
    with torch.cuda.stream(st):
        g.replay()


fl = torch.zeros(128 << 20, dtype=torch.float32, device="cuda")
res = {"graph_warm": timed_steps(graph_run, steps, st, None) * 1e3,
       "single_warm": sum(timed_steps(lambda _: step(0), 1, st, None) for _ in range(steps)) / steps * 1e3,
       "single_flushed": timed_steps(step, steps, st, fl) * 1e3}
# empty-kernel floor: a 1-element torch op bracketed the same way
z = torch.zeros(1, device="cuda")
res["torch_tiny_op_flushed"] = timed_steps(lambda i: z.add_(1), steps, st, fl) * 1e3
print(w, {k: round(v, 2) for k, v in res.items()}, "us")
