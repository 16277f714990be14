#!/usr/bin/env python
"""Summarise an `ncu --set full` report (read here, no GPU needed) into the counters DESIGN.md cites.

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--traffic-key KEY]
With --traffic-key, also records dram read+write bytes per launch into profiles/ncu_traffic.json
(bench.py reports it as roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
]
STALLS = "smsp__average_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name[:120]}")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w:70s} {vals[i]:>16s} {units[i]}")
        st = [(h, vals[i]) for i, h in enumerate(hdr) if h.startswith(STALLS) and h.endswith("per_issue_active.ratio")]
        st = sorted(((float(v), h[len(STALLS):-len("_per_issue_active.ratio")]) for h, v in st if v), reverse=True)
        print("  top stalls (warps per issue):", ", ".join(f"{n}={v:.2f}" for v, n in st[:6]))

        def num(m):
            i = hdr.index(m)
            v = float(vals[i].replace(",", ""))
            u = units[i]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        print(f"  traffic (dram read+write bytes per launch): {traffic:.6e}")
        if key:
            p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
            d = json.load(open(p)) if os.path.exists(p) else {}
            d[key] = traffic
            json.dump(d, open(p, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
