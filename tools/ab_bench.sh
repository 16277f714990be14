#!/bin/bash
# A/B alternative builds on full bench lines: tools/ab_bench.sh <workload> <steps> lib1.so lib2.so ...
w=$1; n=$2; shift 2
for lib in "$@"; do
  cp $lib paper_2603_11504_b200/liblongflow.so
  python bench.py --workload $w --steps $n --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$w', '$lib', 'lat_us %.2f'%d['latency_us'], 'frac %.3f'%d['roofline']['frac'], 'e2e_us %.1f'%(d['e2e']['ms_per_step']*1e3), d['clocks']['sm_mhz'])"
done
