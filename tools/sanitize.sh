#!/bin/bash
# compute-sanitizer passes over the GPU parity tests (run on the GPU box); logs -> gpurun_out/sanitizer_*.log
S=/usr/local/cuda/bin/compute-sanitizer
sel_mem="random_shapes or empty_cache or solo_then_split or gqa_worked or deferred or snapkv or diag"
sel_race="gqa_worked or empty_cache or B2_Hq8_Hkv4 or snapkv"
for tool in memcheck racecheck synccheck; do
  sel=$sel_mem; [ $tool != memcheck ] && sel=$sel_race
  timeout 1200 $S --tool $tool --error-exitcode 9 python -m pytest tests -m gpu -x -q -k "$sel" \
    > gpurun_out/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$tool.log
  tail -3 gpurun_out/sanitizer_$tool.log
done
