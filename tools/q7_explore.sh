#!/bin/bash
# q7 (configs[1]) per-layer-call latency over plan families: split_tokens x k x latency variant
for st in 128 256 512; do for k in 1 2; do for lat in on off; do
  r=$(python bench.py --workload q7 --steps 100 --warmup 5 --no-cpu-baseline --split-tokens $st --ctas-per-sm $k \
      --latency-variant $lat 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f' % d['latency_us'])" 2>/dev/null)
  echo "split_tokens=$st k=$k lat=$lat us=$r"
done; done; done
