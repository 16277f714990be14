"""Debug: pattern of the 1-GPU vs shard difference inside differing units."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from lf_synth import Workload
from tests.test_gpu_plans import _shard_run

tag, B, Hq, Hkv, N, P, od = ("r", 256, 32, 8, 8192, 8, "f32")
G = Hq // Hkv
wl = Workload(tag, B, Hq, Hkv, 128, N, 0, 1)
res, views, plans = _shard_run(wl, P, 1, seed=7, out_dtype=od)
f, s = res[0]
out_f, out_s = f[0].view(B, Hkv, G, 128), s[0].view(B, Hkv, G, 128)
sc_f, sc_s = f[2], s[2]
du = (out_f != out_s).any(-1).any(-1)   # [B][Hkv]
units = du.flatten().nonzero().flatten().tolist()
print("differing units", len(units), "first", units[:10])
for u in units[:6]:
    b, h = divmod(u, Hkv)
    do = (out_f[b, h] != out_s[b, h])
    print(f"unit {u}: out heads differing {do.any(-1).tolist()}, elems {int(do.sum())}")
    ds = (sc_f[b, h] != sc_s[b, h])
    idx = ds.nonzero().flatten()
    print(f"   scores differing {int(ds.sum())} of {N}: first half {int(ds[:4096].sum())} second half {int(ds[4096:].sum())}")
    r = (sc_f[b, h] / sc_s[b, h])
    print(f"   score ratio full/shard: min {float(r.min()):.9f} max {float(r.max()):.9f}")
# match pattern by local unit index within shards
Bs = B // P
loc = torch.zeros(Bs * Hkv, dtype=torch.int32)
for u in units:
    loc[u % (Bs * Hkv)] += 1
print("count of differing per local unit index (over shards):", loc.tolist())
shard_of = [u // (Bs * Hkv) for u in units]
print("per shard:", [shard_of.count(i) for i in range(P)])
