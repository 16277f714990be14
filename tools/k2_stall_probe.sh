#!/bin/bash
# Is the sweep stall tied to the doubled k=2 grids?  The stalling rows, 4 times with and without
# the doubling, one process per row with a 100 s timeout.
for i in 1 2 3 4; do
  for v in "X=1" "LF_NO_K2_DOUBLE=1"; do
    env $v timeout 300 python tools/sweep.py --per-row 100 --out /tmp/k2.jsonl --budgets 512,1024 --batches 32,64,128,256 2> /tmp/k2.err > /dev/null
    echo "run $i $v: points $(wc -l < /tmp/k2.jsonl) $(grep -c 'timed out' /tmp/k2.err) rows timed out"
  done
done
