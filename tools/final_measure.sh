#!/bin/bash
# final validation + bench lines of the round (run on the GPU box); the budget sweep last
tag=${1:-v10}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 300 python bench.py > gpurun_out/${tag}_bench_r.json 2> gpurun_out/${tag}_bench_r.err
timeout 300 python bench.py --workload q7 > gpurun_out/${tag}_bench_q7.json 2>/dev/null
timeout 1200 python tools/sweep.py --out gpurun_out/sweep_${tag}.jsonl > gpurun_out/sweep_${tag}.log 2>&1
