for w in sweep_b8_n512 sweep_b32_n512 q7 sweep_b1_n2048; do
 for e in "" "LF_NO_SPEC=1"; do
  env $e python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$w', '$e', 'S', c['splits'], 'lat_us %.2f'%d['latency_us'])"
 done
done
