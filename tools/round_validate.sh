#!/bin/bash
# Round validation on one B200: GPU suite, smoke, bench lines (ours + the oracle reference arm), a
# 2-rank torchrun functional check on the shared GPU, and the configs[4] sweep in ONE process.
# usage: bash tools/round_validate.sh <tag>   (writes gpurun_out/<tag>_*)
T=${1:-r2}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/${T}_pytest_gpu.log 2>&1
for w in r q7 q3 f1 tiny; do
  python bench.py --workload $w > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err
done
timeout 600 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
LF_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29531 bench.py --gpus 2 --steps 20 --warmup 3 --cpu-seconds 2 > gpurun_out/${T}_bench_2rank_shared.json \
    2> gpurun_out/${T}_bench_2rank_shared.err
timeout 3000 python tools/sweep.py --out gpurun_out/${T}_sweep.jsonl > gpurun_out/${T}_sweep.log 2>&1
echo "sweep rc=$? points $(wc -l < gpurun_out/${T}_sweep.jsonl)" >> gpurun_out/${T}_sweep.log
