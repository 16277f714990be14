for pl in "16,2,0" "16,1,0" "8,2,0" "8,1,0" "4,1,0" "4,2,0"; do
  LF_FORCE_PLAN=$pl python bench.py --workload q7 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$pl', 'S', c['splits'], 'lat_us %.2f'%d['latency_us'])"
done
