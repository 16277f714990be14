#!/bin/bash
# Interleaved A/B of library builds via LF_LIB (run on the GPU box):
#   tools/ab_env.sh "<workloads>" <reps> lib1.so lib2.so ...
ws=$1; reps=$2; shift 2
for r in $(seq $reps); do
  for w in $ws; do
    for lib in "$@"; do
      LF_LIB=$lib python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$w', '$lib', 'lat_us %.2f'%d['latency_us'], 'frac %.3f'%d['roofline']['frac'], 'mhz', d['clocks']['sm_mhz'])"
    done
  done
done
