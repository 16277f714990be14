#!/bin/bash
# Round-end measurement set (run on the GPU box): bench lines for every workload, the reference
# (oracle) arm, the budget sweep, and ncu launch list + full capture of the q7 step.
tag=${1:-v9}
set -x
python bench.py > gpurun_out/${tag}_bench_r.json 2> gpurun_out/${tag}_bench_r.err
for w in q7 q3 f1 tiny; do timeout 300 python bench.py --workload $w > gpurun_out/${tag}_bench_$w.json 2>/dev/null; done
timeout 300 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2>/dev/null
timeout 2400 python tools/sweep.py --out gpurun_out/sweep_${tag}.jsonl > gpurun_out/sweep_${tag}.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_decode -c 300 --csv --log-file gpurun_out/${tag}_launches_q7.csv python bench.py --workload q7 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_decode -s 20 -c 1 -o gpurun_out/${tag}_q7_full python bench.py --workload q7 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_q7.log 2>&1
