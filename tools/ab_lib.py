"""A/B two builds of liblongflow.so on the same box: alternates LF_LIB between them, one bench.py
process per run, R rounds per workload; prints the median latency of each.
usage: python tools/ab_lib.py --libs new.so,old.so --workloads q3,f1,sweep_b64_n2048 [--rounds 3]"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--libs", required=True)
ap.add_argument("--workloads", default="q3,f1")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--extra", default="")
args = ap.parse_args()
libs = args.libs.split(",")
for w in args.workloads.split(","):
    res = {lib: [] for lib in libs}
    for _ in range(args.rounds):
        for lib in libs:
            env = dict(os.environ, LF_LIB=os.path.abspath(lib))
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", w, "--steps", str(args.steps),
                   "--warmup", "5", "--no-cpu-baseline"] + args.extra.split()
            r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                res[lib].append((d["latency_us"], d["clocks"]["sm_mhz"]))
            except Exception:
                print("failed", lib, w, r.stderr[-500:], flush=True)
    for lib in libs:
        v = res[lib]
        if v:
            print(f"{w:22s} {os.path.basename(lib):18s} median {statistics.median(x for x, _ in v):9.2f} us  "
                  f"runs {[round(x, 2) for x, _ in v]}  MHz {[c for _, c in v]}", flush=True)
