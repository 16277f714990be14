S=/usr/local/cuda/bin/compute-sanitizer
run() { echo "== $*"; timeout 600 $S --tool synccheck python tools/dbg/one_step.py "$@" 2>&1 | grep -E "ERROR SUMMARY|^ok|Missing|illegal" | sort | uniq -c | head -5; }
run 1 28 4 2048 0 0 0 3          # q7 default plan
run 40 28 4 2011 128 2 2 3      # plan_family 16-2 lat on, many units per CTA
run 40 28 4 2011 128 2 1 3      # 16-2 lat off
run 20 28 4 2011 128 1 2 3      # 16-1 lat on
run 64 32 8 475 256 2 2 3       # S=2 k=2 lat on
run 64 32 8 475 256 2 1 3       # S=2 k=2 lat off
