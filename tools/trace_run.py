"""Debug: run one decode step of a bench workload with the -DLF_TRACE build and summarise the
per-unit event timeline (ns).  usage: LF_LIB=altlib/lib_trace.so python tools/trace_run.py r"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import workload_of
from lf_synth import Synth, random_cache
from paper_2603_11504_b200 import Cache

w = sys.argv[1] if len(sys.argv) > 1 else "r"
wl = workload_of(w)
split = int(sys.argv[sys.argv.index("--split") + 1]) if "--split" in sys.argv else 0
cache = Cache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N, out_dtype="bf16", split_tokens=split)
plan = cache.plan()
K, V, nv = cache.views()
k0, v0 = random_cache(wl.B, wl.Hkv, wl.N, wl.d, device="cuda")
K.copy_(k0); V.copy_(v0); nv.fill_(wl.N)
del k0, v0
syn = Synth(wl, device="cuda")
q, kn, vn = syn.step()
out, slot, _ = cache.new_outputs()
ctas = 148 * 4
tr = torch.zeros(ctas * 64 * 32, dtype=torch.int64, device="cuda")
for i in range(3):
    cache.decode_step(q, kn, vn, out, slot)
cache.set_trace(tr)
if "--flush" in sys.argv:   # cold L2 / TLB, as bench.py times L2-resident configs
    fl = torch.zeros(128 << 20, dtype=torch.float32, device="cuda")
    fl.amax()
# --b2b K: K back-to-back steps without a sync (PDL overlaps each step's prologue with the previous
# step); the trace keeps the events of the last one (every step writes the same slots)
b2b = int(sys.argv[sys.argv.index("--b2b") + 1]) if "--b2b" in sys.argv else 1
for _ in range(b2b):
    cache.decode_step(q, kn, vn, out, slot)
torch.cuda.synchronize()
a = tr.view(ctas, 64, 32).cpu().numpy().astype(np.int64)
raw0 = a[0, 0, :31].copy()   # CTA 0, first item: raw SM cycles (clock granularity check)
rv = raw0[raw0 > 0]
print("CTA 0 raw cycle offsets from entry:", sorted((rv - a[0, 0, 16]).tolist()))
# events are SM cycles; row 0 slot 16 = entry cycles, slot 31 = entry globaltimer (ns)
ghz = float(os.environ.get("LF_TRACE_GHZ", "1.965"))
for c in range(ctas):
    if a[c, 0, 16] <= 0:
        continue
    clk0, gt0 = a[c, 0, 16], a[c, 0, 31]
    a[c, 0, 31] = 0
    m = a[c] > 0
    a[c][m] = gt0 + np.round((a[c][m] - clk0) / ghz).astype(np.int64)
np.save(f"gpurun_out/trace_{w}.npy", a)
used = a[:, :, 0] > 0
t0 = a[used][:, 0].min()
print("plan", plan, "ctas with events", int(used.any(axis=1).sum()))
names = ["start", "maxdone", "Vdone", "xready", "keypush", "fin", "prodQ", "mmaQ", "xfree", "ofull",
         "ostage", "pushed", "MZ", "comb", "r0done", "xsdone", "Vland", "entry", "csync", "pdlw"] + [""] * 12
rows = a[used].astype(np.float64)
for i, j in [(6, 7), (6, 0), (0, 15), (15, 1), (1, 2), (2, 8), (8, 9), (9, 10), (10, 11), (11, 3), (3, 12),
             (12, 4), (4, 13), (13, 14)]:
    ok = (rows[:, j] > 0) & (rows[:, i] > 0)
    d = rows[ok, j] - rows[ok, i]
    if not ok.any():
        continue
    print(f"{names[i]}->{names[j]}: mean {d.mean()/1e3:.2f} us  p50 {np.median(d)/1e3:.2f}  max {d.max()/1e3:.2f}")
# absolute timeline of the first unit of every CTA (us from the earliest event)
first = a[:, 0].astype(np.float64)
fu = first[(first[:, 6] > 0)]
fu[:, 16] = first[(first[:, 6] > 0), 5]  # V landed (slot 5)
fu[:, 17:20] = first[(first[:, 6] > 0), 16:19]
tmin = fu[fu > 0].min()
print("first unit, us after the earliest event (min / mean / max over CTAs):")
for j in [17, 18, 19, 6, 7, 0, 15, 1, 16, 2, 8, 9, 10, 11, 3, 12, 4, 13, 14]:
    v = fu[fu[:, j] > 0, j] - tmin
    if len(v):
        print(f"  {names[j]:8s} {v.min()/1e3:6.2f} {v.mean()/1e3:6.2f} {v.max()/1e3:6.2f}")
last = np.array([r[r > 0].max() for r in a[used].astype(np.float64)])
print(f"kernel event span {(last.max() - tmin)/1e3:.2f} us")
per_cta = []
for c in range(ctas):
    u = np.nonzero(used[c])[0]
    if len(u) < 2:
        continue
    per_cta.append(a[c, u].astype(np.float64))
if per_cta:
    gaps = np.concatenate([ev[1:, 0] - ev[:-1, 14] for ev in per_cta])
    print(f"r0done(u) -> start(u+1): mean {gaps.mean()/1e3:.2f} us")
    unit = np.concatenate([ev[1:, 0] - ev[:-1, 0] for ev in per_cta])
    print(f"unit period: mean {unit.mean()/1e3:.2f} us  p50 {np.median(unit)/1e3:.2f}")
# per-CTA timeline of the first item relative to the CTA's own PDL wait (cycle-accurate: SM clock)
rel_names = {16: "entry", 17: "csync", 18: "pdlw", 19: "pdlw(softmax)", 20: "sm_base", 21: "sm_n_loaded",
             22: "prod_n_loaded", 24: "prod_qfree", 6: "prodQ", 7: "mmaQ", 0: "start", 15: "xsdone",
             1: "maxdone", 5: "Vland", 2: "Vdone", 8: "xfree", 9: "ofull", 10: "ostage", 11: "pushed",
             3: "xready", 12: "MZ", 4: "keypush", 13: "comb", 14: "r0done", 30: "kdone_seen", 23: "m_ready",
             25: "S_loaded(V)", 26: "P_stored", 27: "P_fenced", 28: "mma_PREADY", 29: "mma_PV_committed"}
r0 = a[used[:, 0], 0].astype(np.float64)
ok0 = r0[:, 18] > 0
print("first item, us after the CTA's own PDL wait (mean over CTAs):")
for j, nm in sorted(rel_names.items(), key=lambda kv: np.mean(r0[ok0 & (r0[:, kv[0]] > 0), kv[0]] - r0[ok0 & (r0[:, kv[0]] > 0), 18]) if (ok0 & (r0[:, kv[0]] > 0)).any() else 1e18):
    m = ok0 & (r0[:, j] > 0)
    if m.any():
        print(f"  {nm:16s} {np.mean(r0[m, j] - r0[m, 18]) / 1e3:7.3f}  ({np.mean(r0[m, j] - r0[m, 18]) * ghz:7.0f} cycles)")
