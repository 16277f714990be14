#!/bin/bash
# compute-sanitizer passes over the GPU parity tests (run on the GPU box); logs -> gpurun_out/sanitizer_*.log
S=/usr/local/cuda/bin/compute-sanitizer
sel_mem="(random_shapes and not bf16) or empty_cache or solo_then_split or gqa_worked or deferred or snapkv or diag or (plan_family and (5-2 or 16-2 or 3-1)) or (sharded and small)"
sel_race="gqa_worked or empty_cache or B2_Hq8_Hkv4 or B1_Hq10 or snapkv or (plan_family and 16-2-off-on)"
for tool in ${TOOLS:-memcheck racecheck synccheck}; do   # one tool per gpurun call (the recipe)
  sel=$sel_mem; [ $tool != memcheck ] && sel=$sel_race
  timeout 1200 $S --tool $tool --error-exitcode 9 python -m pytest tests -m gpu -x -q -k "$sel" \
    > gpurun_out/${TAG:-r2}_sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG:-r2}_sanitizer_$tool.log
  tail -3 gpurun_out/${TAG:-r2}_sanitizer_$tool.log
done
