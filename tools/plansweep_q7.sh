# q7 (configs[1]) latency per forced plan family: S CTAs per unit (split_tokens = 2048 / S), k CTAs per SM.
for pl in "16 2" "16 1" "8 2" "8 1" "4 1" "4 2"; do
  set -- $pl
  python bench.py --workload q7 --steps 100 --warmup 5 --no-cpu-baseline --split-tokens $((2048 / $1)) \
      --ctas-per-sm $2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('S=$1 k=$2', 'S', c['splits'], 'lat_us %.2f'%d['latency_us'])"
done
