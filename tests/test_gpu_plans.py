"""The tcgen05 kernel's plan families against the oracle, shard invariance (multi-GPU correctness by
construction), and liveness of every plan family.

Plan family = (S CTAs per unit, k CTAs per SM, whole-unit "solo" rounds, latency variant); the plan
overrides of lf_cache_config force each one.  Tolerances: tests/parity.py (R12).
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from lf_synth import Synth, Workload, random_cache
from tests.parity import run_lockstep, setup_pair

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cases():
    out = []
    for S in (1, 2, 3, 4, 5, 6, 8, 16):
        for k in (1, 2):
            for solo in ((False,) if S == 1 else (False, True)):
                for lat in ((False,) if S == 1 else (False, True)):
                    chunk = 128 if S == 16 else 256
                    if solo and k == 2 and S * chunk > 1920:   # a k=2 CTA holds <= 1920 tokens
                        continue
                    out.append((S, k, solo, lat))
    return out


@pytest.mark.parametrize("S,k,solo,lat", _cases(),
                         ids=lambda v: str(v) if not isinstance(v, bool) else ("on" if v else "off"))
def test_plan_family_lockstep(cuda_lib, S, k, solo, lat):
    """Every plan family on a shape where each persistent CTA walks several units (>= 2, >= 4 for
    k=2 split plans), with a ragged last chunk, a fill step then evictions: out, scores, slots and
    the cache match the oracle at every step."""
    from paper_2603_11504_b200 import Cache
    chunk = 128 if S == 16 else 256
    N = S * chunk - (37 if S > 1 else 0)
    Hq, Hkv = (32, 8) if (S + k) % 2 == 0 else (28, 4)
    kw = dict(split_tokens=chunk, ctas_per_sm=k, solo=solo, latency_variant=lat)
    probe = Cache(1024 // Hkv, Hq, Hkv, 128, N, **kw)   # 1024 units: enough for a solo round
    C = probe.plan()["clusters"]
    probe.close()
    if solo:   # one round of whole units on every CTA plus a split tail of 37 units
        units = C * S + 37
    else:
        units = (4 if k == 2 else 2) * C + 3
    B = -(-units // Hkv)
    wl = Workload("plan", B, Hq, Hkv, 128, N, N - 1, 3)
    cache, orc, syn = setup_pair(wl, seed=S * 100 + k * 10 + solo * 2 + lat, nthreads=8, **kw)
    plan = cache.plan()
    assert plan["kernel"] == "tcgen05" and plan["splits"] == S, plan
    assert plan["tmem_cols"] == (512 if k == 1 else 256), plan
    assert (plan["solo_rounds"] > 0) == solo, plan
    assert plan["latency_variant"] == int(lat and S > 1), plan
    st = run_lockstep(cache, orc, syn, wl.steps)
    assert st.evictions == 2 * B * Hkv and st.max_out_err < 1e-4, (plan, st)


# Latency-regime plans (steps below 64 MB) the planner's fitted latency model must pick: the best
# measured plan of each point in profiles/r02_lat_explore2.jsonl (B, Hq, Hkv, N) -> (S, split_tokens,
# CTAs per SM, latency variant)
LATENCY_PICKS = [
    ((1, 28, 4, 2048), (16, 128, 2, 1)),   # configs[1] (q7)
    ((2, 32, 8, 512), (4, 128, 2, 1)),     # round 1 kept this on whole units: 10.3 -> 6.6 us
    ((1, 32, 8, 1024), (8, 128, 2, 1)),
    ((4, 32, 8, 1024), (4, 256, 2, 1)),
    ((16, 32, 8, 512), (2, 256, 2, 1)),
]


@pytest.mark.parametrize("shape,pick", LATENCY_PICKS, ids=lambda v: "x".join(map(str, v)))
def test_latency_regime_auto_plan(cuda_lib, shape, pick):
    """The automatic plan of small steps is the measured-best family, and it matches the oracle."""
    from paper_2603_11504_b200 import Cache
    B, Hq, Hkv, N = shape
    c = Cache(B, Hq, Hkv, 128, N)
    plan = c.plan()
    c.close()
    got = (plan["splits"], plan["split_tokens"], 2 if plan["tmem_cols"] == 256 else 1, plan["latency_variant"])
    assert plan["kernel"] == "tcgen05" and got == pick, plan
    wl = Workload("lat", B, Hq, Hkv, 128, N, N - 1, 3)
    cache, orc, syn = setup_pair(wl, seed=B * 7 + N, nthreads=8)
    st = run_lockstep(cache, orc, syn, wl.steps)
    assert st.evictions == 2 * B * Hkv and st.max_out_err < 1e-4, (plan, st)


def _shard_run(wl, P, steps, seed, out_dtype, plan_shards=0, **kw):
    """Steps the whole batch on one cache and, on the same GPU, P shard caches of B/P sequences
    each (plan_batch = B, seq_offset = r B/P; both with the same plan_shards), on the same inputs.
    Returns per-step (out, slot, scores) of both and the final caches."""
    from paper_2603_11504_b200 import Cache
    B, Bs = wl.B, wl.B // P
    K0, V0 = random_cache(B, wl.Hkv, wl.N, wl.d, seed=seed, device="cuda")
    syn = Synth(wl, seed=seed, device="cuda")
    inputs = [syn.step() for _ in range(steps)]
    caches = [Cache(B, wl.Hq, wl.Hkv, wl.d, wl.N, out_dtype=out_dtype, plan_shards=plan_shards, **kw)]
    caches += [Cache(Bs, wl.Hq, wl.Hkv, wl.d, wl.N, out_dtype=out_dtype, plan_batch=B, seq_offset=r * Bs,
                     plan_shards=plan_shards, **kw) for r in range(P)]
    rows = [slice(0, B)] + [slice(r * Bs, (r + 1) * Bs) for r in range(P)]
    for c, sl in zip(caches, rows):
        K, V, nv = c.views()
        K.copy_(K0[sl])
        V.copy_(V0[sl])
        nv.fill_(wl.N - 1)   # one append step, then evictions
    del K0, V0
    torch.cuda.synchronize()
    res = []
    for q, kn, vn in inputs:
        step = []
        for c, sl in zip(caches, rows):
            out, slot, scores = c.new_outputs(with_scores=True)
            c.decode_step(q[sl], kn[sl], vn[sl], out, slot, scores)
            step.append((out, slot, scores))
        torch.cuda.synchronize()
        full = step[0]
        shard = tuple(torch.cat([s[i] for s in step[1:]]) for i in range(3))
        res.append((full, shard))
    plans = [c.plan() for c in caches[:2]]
    views = [c.views() for c in caches]
    return res, views, plans


SHARD_CASES = [  # (tag, B, Hq, Hkv, N, P, out_dtype, plan_shards)
    ("q3", 64, 32, 8, 4096, 2, "bf16", 0),     # plan of the whole batch: solo/split boundary inside a shard
    ("q3", 64, 32, 8, 4096, 8, "f32", 0),
    ("q3", 64, 32, 8, 4096, 8, "bf16", 8),     # plan chosen for one of 8 shards (no solo rounds)
    ("small", 8, 32, 8, 2048, 4, "f32", 4),    # machine-leaving grid: latency variant
    ("g7", 16, 28, 4, 1024, 8, "bf16", 0),     # G = 7
    ("r", 256, 32, 8, 8192, 8, "bf16", 8),     # configs[3] at 8 GPUs: bench.py's strong-scaling shards
    ("r", 256, 32, 8, 8192, 2, "bf16", 2),
]


@pytest.mark.parametrize("case", SHARD_CASES, ids=lambda c: f"{c[0]}_B{c[1]}_N{c[4]}_P{c[5]}_{c[6]}_ps{c[7]}")
def test_sharded_equals_one_gpu(cuda_lib, case):
    """P logical shards, run one after another on one GPU with the plan of the global
    problem (plan_batch, seq_offset, plan_shards: what bench.py's ranks do under --scaling strong),
    give out, scores and slots BIT-IDENTICAL to a one-GPU cache of the whole batch with the same
    plan_shards, step after step, and identical caches."""
    tag, B, Hq, Hkv, N, P, out_dtype, ps = case
    wl = Workload(tag, B, Hq, Hkv, 128, N, 0, 4)
    res, views, plans = _shard_run(wl, P, wl.steps, seed=7, out_dtype=out_dtype, plan_shards=ps)
    assert plans[0]["splits"] == plans[1]["splits"] and plans[0]["split_tokens"] == plans[1]["split_tokens"]
    for t, (full, shard) in enumerate(res):
        for a, b, name in zip(full, shard, ("out", "slot", "scores")):
            assert torch.equal(a, b), f"step {t}: {name} differs between the 1-GPU run and {P} shards ({plans})"
    Kf, Vf, nvf = views[0]
    Ks = torch.cat([v[0] for v in views[1:]])
    Vs = torch.cat([v[1] for v in views[1:]])
    assert torch.equal(Kf, Ks) and torch.equal(Vf, Vs)
    assert torch.equal(nvf, torch.cat([v[2] for v in views[1:]]))
    print(f"{case}: plan {plans[0]}")


def test_shard_plan_arguments(cuda_lib):
    from paper_2603_11504_b200 import Cache, LFError
    with pytest.raises(LFError) as e:   # seq_offset without plan_batch
        Cache(4, 8, 2, 128, 256, seq_offset=4)
    assert e.value.status == 1
    with pytest.raises(LFError) as e:   # shard beyond the global batch
        Cache(4, 8, 2, 128, 256, plan_batch=6, seq_offset=4)
    assert e.value.status == 1
    c = Cache(4, 8, 2, 128, 256, plan_batch=8, seq_offset=4)
    assert c.plan()["kernel"] == "tcgen05"
    with pytest.raises(LFError) as e:   # plan_shards plans have no whole-unit rounds
        Cache(4, 8, 2, 128, 256, plan_shards=2, solo=True)
    assert e.value.status == 1
    c = Cache(64, 32, 8, 128, 4096, plan_batch=256, seq_offset=64, plan_shards=4)
    assert c.plan()["solo_rounds"] == 0


LIVENESS = [  # (budgets, batches, ctas_per_sm, split_tokens, solo)
    ("512,1024", "32,64,128,256", 2, 0, "auto"),
    ("512,1024", "64,256", 2, 256, "off"),
    ("1024", "128,256", 2, 256, "on"),
    ("512,1024", "64,256", 1, 128, "off"),
    ("2048", "64,128", 1, 512, "on"),
]


@pytest.mark.parametrize("race", [False, True], ids=["ordered", "racing-caller"])
@pytest.mark.parametrize("case", LIVENESS, ids=lambda c: f"N{c[0]}_B{c[1]}_k{c[2]}_split{c[3]}_solo{c[4]}")
def test_plan_liveness(cuda_lib, case, race):
    """No plan family hangs: L layer caches stepped back to back in one CUDA graph
    (the sweep's launch pattern) with k = 2 CTAs per SM walking >= 4 units each, and other forced
    families, in a subprocess under a timeout.  'racing-caller' also runs the steps on a side stream
    WITHOUT waiting for the default-stream copies that fill the caches -- the round-1 sweep's bug,
    under which each CTA role read n_valid at a different time and the kernel deadlocked; the kernel
    now reads n_valid once per (CTA, unit) and hands it to its roles (NRDY), so even a racing caller
    gets garbage but never a hang."""
    budgets, batches, k, split, solo = case
    cmd = [sys.executable, os.path.join(ROOT, "tools", "hang_diag.py"), "--lib",
           os.path.join(ROOT, "paper_2603_11504_b200", "liblongflow.so"), "--budgets", budgets, "--batches",
           batches, "--replays", "5", "--timeout", "60", "--ctas-per-sm", str(k), "--split-tokens", str(split),
           "--solo", solo] + (["--race"] if race else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, f"rc={r.returncode}\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}"
    assert "STALL" not in r.stdout
