#!/bin/bash
# Round validation on one B200: GPU suite, smoke, bench lines, and the configs[4] sweep in ONE process.
# usage: bash tools/round_validate.sh <tag>   (writes gpurun_out/<tag>_*)
T=${1:-r2}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/${T}_pytest_gpu.log 2>&1
for w in r q7 q3 f1 tiny; do
  python bench.py --workload $w > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err
done
timeout 3000 python tools/sweep.py --out gpurun_out/${T}_sweep.jsonl > gpurun_out/${T}_sweep.log 2>&1
echo "sweep rc=$? points $(wc -l < gpurun_out/${T}_sweep.jsonl)" >> gpurun_out/${T}_sweep.log
