#!/usr/bin/env python
"""Benchmark of the LongFlow fused decode step (BASELINE.json metric) -- one JSON line on rank 0.

  python bench.py [--gpus N --steps K --warmup W --workload r --scaling weak|strong]
  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
         --master-port P bench.py --gpus N ...
  python bench.py --impl reference ...      # the fp64 CPU oracle on the host cores

A "step" is one lf_decode_step over every (sequence, kv head) unit of the rank's shard: the whole
hot path (logits, softmax, PV, LongFlowScore, argmin, in-place eviction) on a FULL static cache,
so every step evicts.  value = tokens/s summed over ranks (one token per sequence per step).
Inputs of 8 pre-generated steps live in HBM; the cache (8.6 GB per GPU for `r`) is far larger
than L2, so no L2 flush is needed between steps.  Caches below FLUSH_BELOW bytes per GPU would sit in
the 126 MB L2 across steps.  For them the bench cycles L = ceil(8 x L2 / cache)
layer caches of the same shape -- like the L layers of a model, each layer's cache is cold in L2 when
its step runs -- in one CUDA graph of K x L back-to-back steps; ms_per_step = time / (K x L).  When L
would exceed MAX_LAYERS (`tiny`), every timed step is instead preceded by an untimed 512 MB read (L2
flush) and bracketed by its own CUDA events; ms_per_step is their mean.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from lf_synth import CONFIGS, Synth, Workload, bits, random_cache, sweep_workload  # noqa: E402

METRIC = "fused decode-step tokens/s (LongFlow attention+score+evict, full static cache)"


def workload_of(tag: str) -> Workload:
    if tag.startswith("sweep"):
        _, b, n = tag.split("_")
        return sweep_workload(int(b[1:]), int(n[1:]))
    return CONFIGS[tag]


def alg_bytes_per_step(wl: Workload, B: int, out_bytes: int) -> int:
    """SURVEY.md 8(d) D.3 per unit: 4Nd (K+V read) + 4d (k*,v* read) + 4d (victim write)
    + 2Gd (q) + G d out_bytes (out) + 4 (slot)."""
    d, N, G = wl.d, wl.N, wl.G
    per_unit = 4 * N * d + 4 * d + 4 * d + 2 * G * d + G * d * out_bytes + 4
    return per_unit * B * wl.Hkv


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profiles(tag: str):
    """dram bytes read+write per launch from the committed `ncu --set full` summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(tag)
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    def __init__(self, device_index: int, period=0.02):
        self.period = period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    from paper_2603_11504_b200 import dist as lfd
    return lfd.env()


# ------------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg / --impl reference): the fp64 oracle as it stands, on host cores
# ------------------------------------------------------------------------------------------------

class OracleSample:
    """The fp64 oracle (as it stands) on a bounded sample of the workload: Bs full-cache
    sequences with all their kv heads, threads = host cores.  Cost is exactly linear in units,
    so a per-step time scales to the full batch by (B_total / Bs)."""

    def __init__(self, wl: Workload, Bs: int, seed: int = 0, nthreads: int = 0):
        import oracle
        self.wl, self.Bs = wl, Bs
        self.cores = nthreads or os.cpu_count() or 1
        self.orc = oracle.OracleCache(Bs, wl.Hq, wl.Hkv, wl.d, wl.N, nthreads=self.cores)
        k, v = random_cache(Bs, wl.Hkv, wl.N, wl.d, seed=seed)
        self.orc.K[...] = bits(k)
        self.orc.V[...] = bits(v)
        self.orc.n_valid[...] = wl.N
        syn = Synth(Workload(wl.tag, Bs, wl.Hq, wl.Hkv, wl.d, wl.N, 0, 8), seed=seed)
        self.pool = [tuple(bits(x) for x in syn.step()) for _ in range(4)]
        self.i = 0

    def step(self) -> float:
        q, kn, vn = self.pool[self.i % len(self.pool)]
        self.i += 1
        t0 = time.perf_counter()
        self.orc.step(q, kn, vn)
        return time.perf_counter() - t0


def oracle_sample(wl: Workload, B_total: int, seconds_per_step: float, seed: int = 0,
                  nthreads: int = 0) -> OracleSample:
    """Grows the sample (x4 sequences at a time, capped at the batch) until one oracle step over
    it takes about `seconds_per_step`."""
    Bs = 1
    smp = OracleSample(wl, Bs, seed, nthreads)
    t = smp.step()
    while t < seconds_per_step / 2 and Bs < B_total:
        Bs = min(B_total, max(Bs + 1, int(Bs * min(4.0, seconds_per_step / max(t, 1e-6)))))
        smp = OracleSample(wl, Bs, seed, nthreads)
        t = smp.step()
    return smp


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def describe(smp: OracleSample, steps: int, B_total: int) -> str:
    return (f"{smp.Bs} of {B_total} sequences x {smp.wl.Hkv} kv heads (full cache N={smp.wl.N}) of workload "
            f"'{smp.wl.tag}', {steps} timed oracle steps on {smp.cores} threads, per-step time scaled "
            f"linearly by {B_total}/{smp.Bs} units to the whole batch")


def timed_oracle(wl: Workload, B_total: int, seconds: float, seed: int, nthreads: int):
    """max(3 steps, `seconds`) of oracle steps on a sample sized to ~seconds/4 per step
    (BASELINE.md section 4).  Returns (tokens/s, threads, sample description, s/step)."""
    smp = oracle_sample(wl, B_total, seconds / 4, seed, nthreads)
    ts, t0 = [], time.perf_counter()
    while len(ts) < 3 or time.perf_counter() - t0 < seconds:
        ts.append(smp.step())
    sps = float(np.median(ts)) * B_total / smp.Bs
    return B_total / sps, smp.cores, describe(smp, len(ts), B_total), sps


def oracle_rate(wl: Workload, B_total: int, seconds: float = 10.0, seed: int = 0) -> dict:
    """cpu_baseline leg: the oracle on all host cores and on one thread, each for max(3 steps,
    `seconds`), extrapolated linearly in units to the whole batch."""
    v, cores, desc, sps = timed_oracle(wl, B_total, seconds, seed, 0)
    v1, _, desc1, sps1 = timed_oracle(wl, B_total, seconds, seed, 1)
    return {"value": v, "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": desc,
            "ms_per_step": sps * 1e3,
            "one_thread": {"value": v1, "unit": "tokens/s", "ms_per_step": sps1 * 1e3, "sample": desc1},
            "cpu_model": cpu_model()}


def run_reference(args, wl, B_total):
    """--impl reference: the oracle on the host cores, same workload/metric/unit as our arm;
    each step is a bounded sample so the whole W+K run stays within a few minutes."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    per_step = max(0.05, min(args.ref_seconds, 150.0 / (args.steps + args.warmup)))
    smp = oracle_sample(wl, B_total, per_step, args.seed)
    for _ in range(args.warmup):
        smp.step()
    ts = [smp.step() for _ in range(args.steps)]
    sps = float(np.median(ts)) * B_total / smp.Bs
    value = B_total / sps
    desc = describe(smp, args.steps, B_total)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sps * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args, wl, B_total, None),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": smp.cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


FLUSH_BELOW = 1 << 30     # cache bytes per GPU under which part of the cache could stay L2-resident across steps
CYCLE_FACTOR = 8          # cycled layer caches total >= 8 x L2 (4 x left part of a 268 MB cache in L2)
L2_BYTES = 126 << 20
MAX_LAYERS = 256


def layers_for(cb):
    """Layer caches to cycle so that their total is >= 8 x L2 (0: use the flush method)."""
    if cb >= FLUSH_BELOW:
        return 1
    L = -(-CYCLE_FACTOR * L2_BYTES // max(cb, 1))
    return L if L <= MAX_LAYERS else 0


def cache_bytes_per_gpu(wl, B):
    return 2 * wl.N * wl.d * 2 * wl.Hkv * B


def l2_note(cb):
    if cb >= FLUSH_BELOW:
        return "inputs larger than L2 (cache {:.2f} GB per GPU > 126 MB L2)".format(cb / 1e9)
    L = layers_for(cb)
    if L:
        return ("{} layer caches of {:.1f} MB cycled back to back in one CUDA graph ({:.0f} MB > 8 x L2): "
                "each step's cache is cold in L2, as in an L-layer model".format(L, cb / 1e6, L * cb / 1e6))
    return ("L2 flushed before every timed step (512 MB read, untimed; cache {:.1f} MB per GPU); "
            "per-step CUDA events, no graph".format(cb / 1e6))


def timed_steps(fn, steps, stream, flush):
    """ms per step of fn(i) on `stream`: one event pair around all steps, or (flush is a buffer)
    an untimed L2 flush before every step and per-step event pairs, summed."""
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn(None)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    sink = torch.empty((), dtype=flush.dtype, device=flush.device)
    with torch.cuda.stream(stream):
        for i in range(steps):
            # 512 MB READ: evicts the cache from L2 and leaves only clean lines (a write-based flush
            # would leave ~126 MB of dirty lines whose write-back the timed step would pay for)
            torch.amax(flush, dim=0, out=sink)
            evs[i][0].record(stream)
            fn(i)
            evs[i][1].record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / steps


def config_of(args, wl, B_total, plan):
    c = {"workload": wl.tag, "global_batch": B_total, "batch_per_gpu": B_total // max(args.gpus, 1),
         "num_q_heads": wl.Hq, "num_kv_heads": wl.Hkv, "head_dim": wl.d, "budget": wl.N,
         "cache": "full (every step evicts)", "out_dtype": args.out_dtype,
         "parallelism": f"dp{args.gpus} by sequence (no collective on the hot path)",
         "l2": l2_note(cache_bytes_per_gpu(wl, B_total // max(args.gpus, 1))),
         "layer_caches": max(layers_for(cache_bytes_per_gpu(wl, B_total // max(args.gpus, 1))), 1)}
    if plan:
        c.update({"kernel": plan["kernel"], "splits": plan["splits"], "split_tokens": plan["split_tokens"],
                  "solo_rounds": plan.get("solo_rounds", 0), "ctas_per_sm": 2 if plan.get("tmem_cols") == 256 else 1,
                  "latency_variant": plan.get("latency_variant", 0)})
        if args.gpus > 1 and args.scaling == "strong":
            c["shard_plan"] = (f"plan chosen for one of {args.gpus} shards and fixed for the global batch "
                               f"(plan_batch, plan_shards): bit-identical to one GPU with the same plan")
    if getattr(args, "mode", "same_step") != "same_step":
        c["mode"] = args.mode
    return c


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="r", help="tiny | q7 | q3 | r | f1 | sweep_b<B>_n<N>")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (BASELINE configs[3]): the workload's batch is sharded by sequence across the "
                         "GPUs, each shard computed exactly as on one GPU (plan_batch); weak: every GPU holds "
                         "the workload's whole batch")
    ap.add_argument("--ctas-per-sm", type=int, default=0, choices=[0, 1, 2], help="plan override (0 = auto)")
    ap.add_argument("--solo", default="auto", choices=["auto", "on", "off"], help="plan override")
    ap.add_argument("--latency-variant", default="auto", choices=["auto", "on", "off"], help="plan override")
    ap.add_argument("--kernel", default="auto", choices=["auto", "simt", "tcgen05"])
    ap.add_argument("--split-tokens", type=int, default=0)
    ap.add_argument("--out-dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--mode", default="same_step", choices=["same_step", "deferred", "deferred_exclude_newest"],
                    help="eviction mode (R1); deferred = Fig. 2 literal (NEXT-f1)")
    ap.add_argument("--no-graph", action="store_true", help="launch steps directly instead of a CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="cpu_baseline: each of the all-cores and one-thread oracle timings runs max(3 steps, this)")
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    ws, rank, local = dist_env()
    if ws != args.gpus and ws > 1:
        print(f"warning: WORLD_SIZE={ws} != --gpus {args.gpus}", file=sys.stderr)
    args.gpus = max(ws, 1) if ws > 1 else args.gpus
    wl = workload_of(args.workload)
    from paper_2603_11504_b200 import dist as lfd
    B, b0, B_total = lfd.shard(wl.B, args.gpus, rank, args.scaling)
    if args.impl == "reference":
        return run_reference(args, wl, B_total)
    if args.gpus > 1 and ws == 1:
        print("--gpus > 1 needs torchrun (one process per GPU)", file=sys.stderr)
        return 2

    from paper_2603_11504_b200 import Cache
    # one process per GPU; LF_BENCH_SHARE_GPU=1 maps every rank to the visible GPUs round-robin and
    # uses gloo (functional check of the multi-rank path on a single-GPU box, not a measurement)
    share = os.environ.get("LF_BENCH_SHARE_GPU") == "1"
    local_dev = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    local = local_dev
    pg = None
    if ws > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        pg = dist

    onoff = {"auto": None, "on": True, "off": False}
    # strong scaling: this rank's shard is computed with the plan of the whole batch (bit-identical
    # to the one-GPU run); weak scaling: every rank holds a whole problem
    shard_kw = (dict(plan_batch=B_total, seq_offset=b0, plan_shards=args.gpus)
                if args.scaling == "strong" and args.gpus > 1 else {})
    cache_kw = dict(out_dtype=args.out_dtype, kernel=args.kernel, split_tokens=args.split_tokens, device=local,
                    mode=args.mode, ctas_per_sm=args.ctas_per_sm, solo=onoff[args.solo],
                    latency_variant=onoff[args.latency_variant], **shard_kw)
    cache = Cache(B, wl.Hq, wl.Hkv, wl.d, wl.N, **cache_kw)
    plan = cache.plan()
    K, V, nv = cache.views()
    k0, v0 = random_cache(B, wl.Hkv, wl.N, wl.d, seed=args.seed, device=dev, b0=b0)
    K.copy_(k0)
    V.copy_(v0)
    nv.fill_(wl.N)
    if args.mode != "same_step":
        cache.pending().zero_()   # every unit full with a pending victim (slot 0) before the first step
    del k0, v0
    syn = Synth(wl, seed=args.seed, device=dev, B=B, b0=b0)
    pool = [syn.step() for _ in range(8)]
    out, slot, _ = cache.new_outputs()
    stream = torch.cuda.Stream(device=dev)
    # L2-resident cache: L layer caches of the same shape, cycled like the layers of a model
    n_layers = layers_for(cache_bytes_per_gpu(wl, B))
    layers = [cache]
    for _ in range(1, max(n_layers, 1)):
        c2 = Cache(B, wl.Hq, wl.Hkv, wl.d, wl.N, **cache_kw)
        K2, V2, nv2 = c2.views()
        K2.copy_(K)
        V2.copy_(V)
        nv2.copy_(nv)
        if args.mode != "same_step":
            c2.pending().zero_()
        layers.append(c2)
    torch.cuda.synchronize(dev)

    def step(i):
        q, kn, vn = pool[i % len(pool)]
        cache.decode_step(q, kn, vn, out, slot, stream=stream)

    def layer_steps(i):   # one decode step of every layer cache (K x L launches per graph)
        q, kn, vn = pool[i % len(pool)]
        for c in layers:
            c.decode_step(q, kn, vn, out, slot, stream=stream)

    # warm-up (W steps), then optionally capture a graph of the K timed steps (launch-bound configs)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    flush = None
    if n_layers == 0:
        flush = torch.zeros(128 << 20, dtype=torch.float32, device=dev)
    elif n_layers > 1:
        for i in range(args.warmup):
            layer_steps(i)
        torch.cuda.synchronize(dev)
    graph = None
    if not args.no_graph and flush is None:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(args.steps):
                layer_steps(i) if n_layers > 1 else step(i)
        torch.cuda.synchronize(dev)
        graph.replay()     # one untimed replay (graph upload)
        torch.cuda.synchronize(dev)

    if pg:
        pg.barrier()
    torch.cuda.synchronize(dev)
    def run_all(i):
        if i is not None:
            step(i)
        elif graph is not None:
            with torch.cuda.stream(stream):
                graph.replay()
        else:
            for j in range(args.steps):
                layer_steps(j) if n_layers > 1 else step(j)

    steps_timed = args.steps * max(n_layers, 1)
    with ClockSampler(local) as clk:
        ms = timed_steps(run_all, steps_timed, stream, flush) * steps_timed
    if pg:
        pg.barrier()
    ms_max = lfd.max_over_ranks(ms, device=dev)
    gather = None
    if pg:
        # off the hot path: gather every rank's out / slot over NCCL (NVLink) and time it
        torch.cuda.synchronize(dev)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        out_all = lfd.gather_rows(out)
        slot_all = lfd.gather_rows(slot)
        g1.record()
        torch.cuda.synchronize(dev)
        gather = {"us": lfd.max_over_ranks(g0.elapsed_time(g1) * 1e3, device=dev),
                  "bytes": out_all.numel() * out_all.element_size() + slot_all.numel() * 4}
    ms_step = ms_max / steps_timed
    value = B_total / (ms_step / 1e3)

    # ---- end to end through the public host API: H2D of the step's inputs + D2H of out/slot
    e2e = None
    q0, kn0, vn0 = pool[0]
    hq = [t.cpu().pin_memory() for t in pool[0]]
    oh = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    sh = torch.empty(slot.shape, dtype=torch.int32).pin_memory()
    e2e_steps = max(10, min(args.steps, 100))
    for _ in range(3):
        cache.decode_step_host(*hq, oh, sh, stream=stream)
    if pg:
        pg.barrier()
    torch.cuda.synchronize(dev)
    def e2e_run(i):   # cycles the layer caches like the timed region (each step's cache cold in L2)
        for j in range(1 if i is not None else e2e_steps):
            layers[j % len(layers)].decode_step_host(*hq, oh, sh, stream=stream)

    e_ms = torch.tensor([lfd.max_over_ranks(timed_steps(e2e_run, e2e_steps, stream, flush), device=dev)])
    h2d = sum(t.numel() * t.element_size() for t in hq)
    d2h = oh.numel() * oh.element_size() + sh.numel() * 4
    e2e = {"value": B_total / (float(e_ms.item()) / 1e3), "unit": "tokens/s",
           "h2d_bytes_per_step": h2d * args.gpus, "d2h_bytes_per_step": d2h * args.gpus,
           "ms_per_step": float(e_ms.item()), "steps": e2e_steps, "api": "lf_decode_step_host",
           "io": ("pinned host buffers: the kernel reads q/k*/v* from and writes out/slot to them over the host "
                  "link inside the timed step (zero-copy), then one stream sync")}

    out_bytes = 2 if args.out_dtype == "bf16" else 4
    alg = alg_bytes_per_step(wl, B, out_bytes)
    peak, peak_src = peaks()
    achieved = alg / (ms_step / 1e3) / 1e9
    traffic = traffic_from_profiles(f"{wl.tag}_B{B}_{plan['kernel']}")
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "latency_us": ms_step * 1e3,
        "steps_per_s": 1e3 / ms_step, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded bf16 N(0,1) K/V, query random walk)",
        "config": config_of(args, wl, B_total, plan),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": f"lf decode ({plan['kernel']})",
                     "alg_bytes_per_launch": alg,
                     "frac_of_nominal_8tbs": achieved / 8000.0},   # north star quotes B200's ~8 TB/s
        "hbm_gbs_aggregate": achieved * args.gpus,
        "e2e": e2e,
        "gpu_launches": steps_timed * cache.kernels_per_step(),
        "clocks": clk.summary(),
        "graph": graph is not None,
    }
    if gather:
        line["nccl_gather_out_slot"] = gather
    if rank == 0 and not args.no_cpu_baseline:   # rank 0 only; the other ranks wait at the barrier below
        line["cpu_baseline"] = oracle_rate(wl, B_total, seconds=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
