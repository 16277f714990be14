#!/bin/bash
# usage: tools/sweep_split.sh <workload> <split_tokens...>   (run on the GPU box)
w=$1; shift
for s in "$@"; do
  python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --split-tokens $s 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
c=d['config']
print('$w', 'split', c['split_tokens'], 'S', c['splits'], 'lat_us %.1f'%d['latency_us'], 'frac %.3f'%d['roofline']['frac'])"
done
