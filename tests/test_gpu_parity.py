"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element.

Run on a B200 via gpurun: ``python -m pytest tests -m gpu``.  Tolerances: tests/parity.py (R12).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from lf_synth import CONFIGS, Synth, Workload, bits, bf16, random_cache
from tests.parity import (Stats, accept_slots, assert_cache_equal, check_out, check_scores, run_lockstep,
                          setup_pair)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
KERNELS = ["simt", "tcgen05"]


def _kernel_ok(kernel, G, d):
    from paper_2603_11504_b200 import LFError, Cache
    try:
        Cache(1, G, 1, d, 256, kernel=kernel).close()
        return True
    except LFError as e:
        if e.status == 2:   # LF_ERR_UNSUPPORTED
            return False
        raise


def _need(kernel, G, d):
    if not _kernel_ok(kernel, G, d):
        pytest.skip(f"{kernel} not built for G={G} d={d}")


# --- configs[0]: tiny, the whole 512-step trajectory --------------------------------------

@pytest.mark.parametrize("out_dtype", ["f32", "bf16"])
def test_tiny_full_trajectory(cuda_lib, out_dtype):
    wl = CONFIGS["tiny"]
    cache, orc, syn = setup_pair(wl, kernel="simt", out_dtype=out_dtype)
    st = run_lockstep(cache, orc, syn, wl.steps, out_dtype=out_dtype, check_cache_every=64)
    assert st.evictions == wl.steps - (wl.N - wl.prefill)
    print(f"tiny {out_dtype}: {st}")


# --- random small shapes: several tiles, ragged tails, splits, fill + evict phases ----------

SHAPES = [  # (B, Hq, Hkv, d, N, prefill, steps, split_tokens)
    (2, 2, 2, 64, 2, 0, 6, 0),          # minimum budget, empty start
    (1, 3, 1, 64, 3, 1, 8, 0),          # G=3, budget 3
    (3, 4, 2, 128, 127, 120, 20, 0),     # ragged single tile
    (2, 8, 4, 128, 129, 129, 12, 128),  # full, 2 splits, 1-token tail split
    (2, 14, 2, 128, 300, 290, 20, 128),  # G=7, 3 splits
    (1, 8, 1, 64, 1000, 995, 12, 256),  # G=8, d=64, 4 splits
    (4, 32, 8, 128, 512, 500, 16, 0),   # Q3-like group structure
    (1, 2, 1, 128, 700, 650, 60, 0),    # G=2 crossing the fill boundary
    (64, 32, 8, 128, 384, 380, 6, 0),   # 512 units: several units per persistent cluster
    (48, 32, 8, 128, 384, 370, 14, 128),  # 384 units x 3-CTA clusters, fill -> evict
    (2, 3, 3, 128, 300, 290, 14, 128),  # G=1 at d=128 (tcgen05 with one live head), 3 splits
    (5, 4, 4, 128, 640, 630, 14, 0),    # G=1, solo units
    (1, 10, 2, 128, 1100, 1090, 14, 384),  # G=5, 3-tile CTAs + ragged last chunk (latency variant)
]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "B{}_Hq{}_Hkv{}_d{}_N{}_p{}".format(*s[:6]))
def test_random_shapes(cuda_lib, kernel, shape):
    B, Hq, Hkv, d, N, pre, steps, split = shape
    _need(kernel, Hq // Hkv, d)
    wl = Workload("rand", B, Hq, Hkv, d, N, pre, steps)
    cache, orc, syn = setup_pair(wl, kernel=kernel, split_tokens=split, seed=B * 31 + N)
    st = run_lockstep(cache, orc, syn, steps)
    assert st.max_out_err < 1e-4, st


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "B{}_Hq{}_Hkv{}_d{}_N{}_p{}".format(*s[:6]))
def test_random_shapes_bf16_out(cuda_lib, kernel, shape):
    """The production output dtype (bf16, the one bench.py times) on every shape and both kernels:
    out within 1 bf16 ulp of RNE(oracle) elementwise (R12), scores and slots as in fp32 mode (Alg. 1
    P:539 o_t <- o_acc / l_acc, rounded once)."""
    B, Hq, Hkv, d, N, pre, steps, split = shape
    _need(kernel, Hq // Hkv, d)
    wl = Workload("rand", B, Hq, Hkv, d, N, pre, steps)
    cache, orc, syn = setup_pair(wl, kernel=kernel, split_tokens=split, seed=B * 37 + N, out_dtype="bf16")
    run_lockstep(cache, orc, syn, steps, out_dtype="bf16")


@pytest.mark.parametrize("kernel", KERNELS)
def test_maximum_budget(cuda_lib, kernel):
    """The largest budget the library builds (65,536 slots, lf_cache_create's limit): full cache,
    lockstep eviction steps (tcgen05 G=4: 16 CTAs x 4,096 tokens per unit; CUDA-core G=1)."""
    Hq = 8 if kernel == "tcgen05" else 2     # the group sizes LF_KERNEL_AUTO routes to each kernel
    _need(kernel, Hq // 2, 128)
    wl = Workload("maxN", 1, Hq, 2, 128, 65536, 65536, 3)
    cache, orc, syn = setup_pair(wl, kernel=kernel, seed=65536)
    st = run_lockstep(cache, orc, syn, wl.steps)
    assert st.evictions == 2 * wl.steps and st.max_out_err < 1e-4, st


@pytest.mark.parametrize("kernel", KERNELS)
def test_tiling_invariance(cuda_lib, kernel):
    """C.3 #15: results do not depend on the split plan (within fp32), and the
    slot is identical unless the oracle sees a near-tie."""
    _need(kernel, 4, 128)
    wl = Workload("tile", 2, 8, 2, 128, 1536, 1536, 10)
    outs = []
    for split in (128, 384, 768, 1536):
        cache, orc, syn = setup_pair(wl, kernel=kernel, split_tokens=split, seed=5)
        assert cache.plan()["split_tokens"] == split
        run_lockstep(cache, orc, syn, wl.steps)
        outs.append(bits(cache.views()[0]))
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])


@pytest.mark.parametrize("kernel", KERNELS)
def test_large_logits_stress(cuda_lib, kernel):
    """R5: logit range ~100 (sigma_s = 12): no Inf/NaN, parity holds (the paper's no-max fp32
    softmax would overflow at s > 88.7)."""
    _need(kernel, 4, 128)
    wl = Workload("stress", 2, 8, 2, 128, 640, 600, 30)
    cache, orc, syn = setup_pair(wl, kernel=kernel, sigma_s=12.0, seed=3, key_outliers=True)
    run_lockstep(cache, orc, syn, wl.steps)


@pytest.mark.parametrize("kernel", KERNELS)
def test_increasing_logits(cuda_lib, kernel):
    """Keys aligned with the query and growing along the slots: every later tile raises the max
    (exercises the max/combination logic across tiles and splits)."""
    _need(kernel, 4, 128)
    B, Hq, Hkv, d, N = 1, 4, 1, 128, 1024
    from paper_2603_11504_b200 import Cache
    cache = Cache(B, Hq, Hkv, d, N, kernel=kernel, split_tokens=256)
    orc = oracle.OracleCache(B, Hq, Hkv, d, N)
    rng = np.random.default_rng(0)
    qdir = rng.standard_normal(d)
    qdir /= np.linalg.norm(qdir)
    ramp = np.linspace(-30, 30, N)[:, None] * qdir[None, :] * math.sqrt(d)   # logits ~ -30 .. 30
    K = bf16(ramp + 0.1 * rng.standard_normal((N, d)))[None]
    V = bf16(rng.standard_normal((N, d)))[None]
    cache.prefill(0, K.cuda(), V.cuda())
    orc.prefill(0, bits(K), bits(V))
    q = bf16(np.tile(qdir, (Hq, 1))[None] * 1.0)
    kn, vn = bf16(rng.standard_normal((1, 1, d))), bf16(rng.standard_normal((1, 1, d)))
    st = Stats()
    out, slot, scores = cache.new_outputs(with_scores=True)
    cache.decode_step(q.cuda(), kn.cuda(), vn.cuda(), out, slot, scores)
    torch.cuda.synchronize()
    o_ref, s_ref, sc_ref = orc.compute(bits(q), bits(kn), bits(vn))
    check_out(out.cpu().double().numpy(), o_ref, "f32", st)
    check_scores(scores.cpu().numpy(), sc_ref, orc.n_valid, st)
    accept_slots(slot.cpu().numpy(), s_ref, sc_ref, orc.n_valid, N, st)


# --- hand-built caches ------------------------------------------------------------------------

def _embed(rows, d):
    a = np.zeros((len(rows), d))
    a[:, :len(rows[0])] = rows
    return a


@pytest.mark.parametrize("kernel,d", [("simt", 64), ("simt", 128), ("tcgen05", 128)])
@pytest.mark.parametrize("out_dtype", ["f32", "bf16"])
def test_gqa_worked_example_on_gpu(cuda_lib, kernel, d, out_dtype):
    """C.3 #7 embedded in d = 64 / 128 (zero padding leaves logits, L1 norms and outputs unchanged);
    at d = 128 it runs on the tcgen05 kernel (G = 2 in the M=128 x N=8 logit MMA).  bf16-out mode
    must give the golden outputs rounded once to bf16."""
    _need(kernel, 2, d)
    from paper_2603_11504_b200 import Cache
    g = json.load(open(os.path.join(GOLD, "gqa_worked_example.json")))
    cache = Cache(1, 2, 1, d, 3, kernel=kernel, softmax_scale=math.log(2.0), out_dtype=out_dtype)
    K = bf16(_embed(g["K"], d))[None].cuda()
    V = bf16(_embed(g["V"], d))[None].cuda()
    cache.prefill(0, K, V)
    q = bf16(_embed(g["q"], d))[None].cuda()
    kn = bf16(_embed([g["k_new"]], d))[None].cuda()
    vn = bf16(_embed([g["v_new"]], d))[None].cuda()
    out, slot, scores = cache.new_outputs(with_scores=True)
    cache.decode_step(q, kn, vn, out, slot, scores)
    torch.cuda.synchronize()
    want = np.asarray(g["out"], dtype=np.float64)
    if out_dtype == "bf16":   # rounded once, RNE (R10/R12): 0.6 -> 0.6015625
        want = torch.tensor(want, dtype=torch.float32).to(torch.bfloat16).double().numpy()
    np.testing.assert_allclose(out[0, :, :2].double().cpu().numpy(), want, rtol=1e-6, atol=1e-6)
    assert float(out[0, :, 2:].float().abs().max()) == 0.0
    np.testing.assert_allclose(scores[0, 0].cpu().numpy(), g["scores"], rtol=1e-6)
    assert int(slot[0, 0]) == g["slot"]
    Kc, Vc, nv = cache.views()
    np.testing.assert_array_equal(Kc[0, 0, :, :2].float().cpu().numpy(), g["K_after"])
    np.testing.assert_array_equal(Vc[0, 0, :, :2].float().cpu().numpy(), g["V_after"])
    assert int(nv[0, 0]) == 3


@pytest.mark.parametrize("kernel", KERNELS)
def test_empty_cache_and_ties(cuda_lib, kernel):
    """n = 0: out = v_new, slot 0 (append).  All-zero V: every score 0 -> slot 0.
    Duplicate minimum tokens -> the lower index (R7)."""
    _need(kernel, 4, 128)
    from paper_2603_11504_b200 import Cache
    d, N = 128, 300
    cache = Cache(1, 4, 1, d, N, kernel=kernel, split_tokens=128)
    rng = np.random.default_rng(1)
    q = bf16(rng.standard_normal((1, 4, d))).cuda()
    kn = bf16(rng.standard_normal((1, 1, d))).cuda()
    vn = bf16(rng.standard_normal((1, 1, d))).cuda()
    out, slot, scores = cache.new_outputs(with_scores=True)
    cache.decode_step(q, kn, vn, out, slot, scores)
    torch.cuda.synchronize()
    assert int(slot[0, 0]) == 0
    np.testing.assert_array_equal(out[0].cpu().numpy(), np.repeat(vn[0].float().cpu().numpy(), 4, axis=0))
    assert torch.isinf(scores).all()
    # all-zero values, full cache
    K = bf16(rng.standard_normal((1, N, d))).cuda()
    cache.prefill(0, K, torch.zeros(1, N, d, dtype=torch.bfloat16, device="cuda"))
    cache.decode_step(q, kn, vn, out, slot, scores)
    torch.cuda.synchronize()
    assert int(slot[0, 0]) == 0 and float(scores[0, 0].abs().max()) == 0.0
    # two identical minimal tokens in different splits -> the lower slot
    Vr = rng.standard_normal((N, d)) * 4
    Kr = rng.standard_normal((N, d))
    for j in (140, 290):
        Vr[j] = 1e-3
        Kr[j] = -1.0
    cache.prefill(0, bf16(Kr)[None].cuda(), bf16(Vr)[None].cuda())
    cache.decode_step(q, kn, vn, out, slot, scores)
    torch.cuda.synchronize()
    assert float(scores[0, 0, 140]) == float(scores[0, 0, 290])
    assert int(slot[0, 0]) == 140


def test_prefill_errors(cuda_lib):
    from paper_2603_11504_b200 import Cache, LFError
    cache = Cache(2, 4, 2, 64, 16)
    k = torch.zeros(2, 17, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(LFError) as e:
        cache.prefill(0, k, k)
    assert e.value.status == 4
    with pytest.raises(LFError) as e:
        cache.prefill(2, k[:, :3], k[:, :3])
    assert e.value.status == 1


@pytest.mark.parametrize("pinned", [True, False], ids=["pinned", "pageable"])
@pytest.mark.parametrize("B,N,mode,out_dtype", [
    (2, 256, "same_step", "f32"),        # small step (pageable: zero-copy through the mapped staging)
    (64, 4096, "same_step", "bf16"),     # large step (pageable: H2D, kernel, D2H) across solo/split units
    (64, 512, "deferred", "f32"),        # deferred mode (pre-pass + kernel)
])
def test_host_entry_point_matches_device(cuda_lib, B, N, mode, out_dtype, pinned):
    """lf_decode_step_host (host buffers: pinned caller buffers are read and written by the kernel
    directly, pageable ones go through the staging) == lf_decode_step on the same inputs, bit for
    bit, and the caches stay equal."""
    from paper_2603_11504_b200 import Cache
    wl = Workload("host", B, 32 if B > 2 else 8, 8 if B > 2 else 2, 128, N, N - 8, 4)

    def make():
        syn = Synth(wl, seed=9)
        c = Cache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N, out_dtype=out_dtype, mode=mode)
        K, V = syn.prefill()
        for b in range(wl.B):
            c.prefill(b, K[b].cuda(), V[b].cuda())
        return c, syn
    c1, syn = make()
    c2, _ = make()
    out, slot, _ = c1.new_outputs()
    for _ in range(wl.steps):
        q, kn, vn = syn.step()
        c1.decode_step(q.cuda(), kn.cuda(), vn.cuda(), out, slot)
        oh = torch.empty(out.shape, dtype=out.dtype)
        sh = torch.empty(slot.shape, dtype=torch.int32)
        hin = (q, kn, vn)
        if pinned:
            oh, sh = oh.pin_memory(), sh.pin_memory()
            hin = tuple(t.pin_memory() for t in hin)
        c2.decode_step_host(*hin, oh, sh)
        torch.cuda.synchronize()
        assert torch.equal(oh, out.cpu())
        np.testing.assert_array_equal(sh.numpy(), slot.cpu().numpy())
    for a, b in zip(c1.views(), c2.views()):
        assert torch.equal(a, b)


def test_library_owned_slab_and_determinism(cuda_lib):
    from paper_2603_11504_b200 import Cache
    wl = Workload("det", 3, 8, 2, 128, 700, 700, 3)
    syn = Synth(wl, seed=2)
    K, V = syn.prefill()
    res = []
    for owned in (True, False, False):
        c = Cache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N, library_owned=owned)
        for b in range(wl.B):
            c.prefill(b, K[b].cuda(), V[b].cuda())
        out, slot, scores = c.new_outputs(with_scores=True)
        s2 = Synth(wl, seed=2)
        for _ in range(wl.steps):
            q, kn, vn = s2.step()
            c.decode_step(q.cuda(), kn.cuda(), vn.cuda(), out, slot, scores)
        torch.cuda.synchronize()
        res.append((out.cpu(), slot.cpu(), scores.cpu()))
        c.close()
    for r in res[1:]:
        for a, b in zip(r, res[0]):
            assert torch.equal(a, b)


# --- configs[1]: Q7, single sequence 28/4 --------------------------------------------------

def test_q7_lockstep_1000_steps(cuda_lib):
    wl = CONFIGS["q7"]
    cache, orc, syn = setup_pair(wl, nthreads=4)
    st = run_lockstep(cache, orc, syn, 1000, check_cache_every=250)
    print(f"q7 1000 steps: {st}")


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("LF_SLOW"), reason="set LF_SLOW=1 (several minutes of oracle time)")
def test_q7_full_trajectory(cuda_lib):
    """All 10,240 tokens of configs[1] (prefill 512 + 9,728 decode steps), lockstep."""
    wl = CONFIGS["q7"]
    cache, orc, syn = setup_pair(wl, nthreads=8)
    st = run_lockstep(cache, orc, syn, wl.steps, with_scores=False, check_cache_every=1000)
    print(f"q7 full: {st}")


# --- full-size configs in the bench's launch configuration: sampled units ---------------------

@pytest.mark.parametrize("out_dtype", ["f32", "bf16"])
@pytest.mark.parametrize("tag", ["q3", "r"])
def test_full_size_sampled_units(cuda_lib, tag, out_dtype):
    """BASELINE configs[2]/[3] at full size, cache full (steady state), the plan and output dtype
    bench.py uses (bf16): every unit is checked for the one-slot-changes invariant; 12 sampled units
    are checked element by element against the oracle (their K/V/q come from the seeded generator)."""
    from paper_2603_11504_b200 import Cache
    wl = CONFIGS[tag]
    cache = Cache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N, out_dtype=out_dtype)
    K, V, nv = cache.views()
    k0, v0 = random_cache(wl.B, wl.Hkv, wl.N, wl.d, seed=11, device="cuda")
    K.copy_(k0)
    V.copy_(v0)
    nv.fill_(wl.N)
    del k0, v0
    syn = Synth(wl, seed=11, device="cuda")
    q, kn, vn = syn.step()
    K_before = K.clone()
    rng = np.random.default_rng(0)
    units = [(int(b), int(h)) for b, h in zip(rng.integers(0, wl.B, 12), rng.integers(0, wl.Hkv, 12))]
    host = {u: (bits(K[u]), bits(V[u])) for u in units}
    out, slot, scores = cache.new_outputs(with_scores=True)
    cache.decode_step(q, kn, vn, out, slot, scores)
    torch.cuda.synchronize()
    # every unit: exactly the victim row changed, and it now holds (k*, v*)
    changed = (K != K_before).any(dim=-1)
    del K_before
    sl = slot.long()
    assert int(changed.sum()) <= wl.B * wl.Hkv
    assert not bool((changed & ~torch.nn.functional.one_hot(sl, wl.N).bool()).any())
    rows_k = torch.gather(K, 2, sl[:, :, None, None].expand(-1, -1, 1, wl.d))[:, :, 0]
    assert torch.equal(rows_k, kn)
    assert bool(torch.isfinite(scores).all()) and bool((sl >= 0).all() and (sl < wl.N).all())
    qh, knh, vnh = bits(q), bits(kn), bits(vn)
    st = Stats()
    for (b, h) in units:
        Kb, Vb = host[(b, h)]
        r = oracle.unit_attend(qh[b, h * wl.G:(h + 1) * wl.G], Kb, Vb, knh[b, h], vnh[b, h])
        check_out(out[b, h * wl.G:(h + 1) * wl.G].cpu().double().numpy(), r["out"], out_dtype, st)
        sc = scores[b, h].cpu().numpy().astype(np.float64)
        assert np.all(np.abs(sc - r["scores"]) <= 1e-4 * r["scores"] + 1e-30)
        s = int(slot[b, h])
        assert s == r["slot"] or r["scores"][s] <= (1 + 1e-4) * r["scores"].min() + 1e-30
    print(f"{tag}: {st}")


def test_solo_then_split_schedule(cuda_lib):
    """A plan with whole-unit (solo) rounds followed by a split tail (B=64, 32/8, N=2048 -> 512
    units over 74 two-CTA clusters): every unit, solo or split, matches the oracle."""
    wl = Workload("mix", 64, 32, 8, 128, 2048, 2040, 4)
    cache, orc, syn = setup_pair(wl, nthreads=8)
    plan = cache.plan()
    if plan["solo_rounds"] == 0:
        pytest.skip(f"planner chose no solo rounds here: {plan}")
    st = run_lockstep(cache, orc, syn, wl.steps)
    print(plan, st)


# --- back-to-back steps with no host synchronisation (PDL overlap + speculative first tiles) ------

def _enqueue_b2b(plan_of_steps, graph):
    """plan_of_steps: list of (cache, q, kn, vn, out, slot) enqueued in order on one stream."""
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for c, q, kn, vn, out, slot in plan_of_steps:
                c.decode_step(q, kn, vn, out, slot, stream=st)
        g.replay()
    else:
        with torch.cuda.stream(st):
            for c, q, kn, vn, out, slot in plan_of_steps:
                c.decode_step(q, kn, vn, out, slot, stream=st)
    torch.cuda.synchronize()


@pytest.mark.parametrize("graph", [False, True], ids=["stream", "graph"])
def test_back_to_back_steps_no_sync(cuda_lib, graph):
    """Full caches stepped back to back on one stream with no host synchronisation (the bench's
    launch pattern): with programmatic dependent launch, step t+1's prologue runs while step t is
    still writing its victim row, and its first dependent read must come after its PDL wait.
    Cache A (the q7 shape: 16-CTA clusters, one tile per CTA, the latency variant) runs 40 steps
    alone, then A and a second cache B (2 x 8/2, N=256, streaming variant) are interleaved
    A B A B ... for 40 more steps each.  Every step's out and slot, and the final caches, must
    equal the oracle run step by step."""
    wa = Workload("b2b_a", 1, 28, 4, 128, 2048, 2048, 0)
    wb = Workload("b2b_b", 2, 8, 2, 128, 256, 256, 0)
    A = setup_pair(wa, seed=5, nthreads=4)
    B = setup_pair(wb, seed=6, nthreads=4)
    order = [A] * 40 + [A, B] * 40
    steps = []
    for cache, orc, syn in order:
        q, kn, vn = syn.step()
        out, slot, _ = cache.new_outputs(with_scores=False)
        steps.append((cache, orc, (q, kn, vn), out, slot))
    _enqueue_b2b([(c, q.cuda(), kn.cuda(), vn.cuda(), out, slot) for c, _, (q, kn, vn), out, slot in steps],
                 graph)
    stats = Stats()
    for cache, orc, (q, kn, vn), out, slot in steps:
        qb, kb, vb = bits(q), bits(kn), bits(vn)
        nv_before = orc.n_valid.copy()
        o_ref, s_ref, sc_ref = orc.compute(qb, kb, vb, want_scores=True)
        check_out(out.cpu().double().numpy(), o_ref, cache.out_dtype, stats)
        chosen = accept_slots(slot.cpu().numpy(), s_ref, sc_ref, nv_before, orc.N, stats)
        orc.apply(kb, vb, chosen)
    assert_cache_equal(A[0], A[1])
    assert_cache_equal(B[0], B[1])
    print(f"back to back ({'graph' if graph else 'stream'}): A plan {A[0].plan()}, B plan {B[0].plan()}, {stats}")
