"""Render a tools/sweep.py jsonl as the markdown table in profiles/.  usage: python tools/sweep_md.py in.jsonl title"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1])]
Ns = sorted({r["N"] for r in rows})
Bs = sorted({r["B"] for r in rows})
d = {(r["B"], r["N"]): r for r in rows}
print(f"# {sys.argv[2] if len(sys.argv) > 2 else 'Budget sweep'}\n")
print("latency per decode step (us) / fraction of the measured HBM copy peak; 32/8 GQA, d=128, full cache, "
      "bf16 out, CUDA graph of back-to-back steps. Unmarked: cache >= 1 GB (far larger than the 126 MB L2). "
      "`L`: cache < 1 GB, L = ceil(8 x L2 / cache) layer caches cycled in the graph so each step's cache is cold "
      "in L2 (SURVEY D.4); the step time is per layer call. `*`: every step timed alone after an untimed 512 MB "
      "read that evicts L2.\n")
print("| B \\ N | " + " | ".join(map(str, Ns)) + " |")
print("|---" * (len(Ns) + 1) + "|")
for B in Bs:
    cells = []
    for N in Ns:
        r = d[B, N]
        star = "*" if "flushed" in r.get("l2", "") else ("L" if r.get("layer_caches", 1) > 1 else "")
        cells.append(f"{r['latency_us']:.1f} / {r['frac_measured_peak']:.2f}{star}")
    print(f"| {B} | " + " | ".join(cells) + " |")
