#!/bin/bash
# ncu evidence of the current kernel (run on the GPU box): launch lists (gpu__time_duration, the
# recipe's --clock-control none pass) of the default bench command, and one `--set full` capture of
# the decode kernel for r, q3, q7, f1 and a k=2 sweep point.  Every command runs once without ncu
# first (the recipe's rule).  usage: bash tools/ncu_round.sh <tag>
T=${1:-r2}
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode -c 40 --csv --log-file gpurun_out/${T}_launches_r.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for w in r q3 q7 f1 sweep_b128_n512 sweep_b32_n8192; do
  extra=""; [ $w = sweep_b128_n512 ] && extra="--ctas-per-sm 2"
  python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-graph $extra > /dev/null 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_decode -s 6 -c 1 \
      -o gpurun_out/${T}_full_$w python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-graph $extra \
      > gpurun_out/${T}_ncu_$w.log 2>&1
done
