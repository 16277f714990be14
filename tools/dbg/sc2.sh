S=/usr/local/cuda/bin/compute-sanitizer
echo "== plain 300 steps"; timeout 300 python tools/dbg/one_step.py 40 28 4 2011 128 2 2 300 2>&1 | tail -2
echo "== memcheck"; timeout 600 $S --tool memcheck python tools/dbg/one_step.py 40 28 4 2011 128 2 2 3 2>&1 | grep -E "ERROR SUMMARY|^ok|Invalid|illegal|at .*tc_decode|Address" | sort | uniq -c | head -12
echo "== synccheck B=4 (1 unit per CTA)"; timeout 600 $S --tool synccheck python tools/dbg/one_step.py 4 28 4 2011 128 2 2 3 2>&1 | grep -E "ERROR SUMMARY|^ok|Missing|illegal" | sort | uniq -c
echo "== synccheck B=8"; timeout 600 $S --tool synccheck python tools/dbg/one_step.py 8 28 4 2011 128 2 2 3 2>&1 | grep -E "ERROR SUMMARY|^ok|Missing|illegal" | sort | uniq -c
echo "== synccheck S=8 k=2 B=40"; timeout 600 $S --tool synccheck python tools/dbg/one_step.py 40 28 4 1011 128 2 2 3 2>&1 | grep -E "ERROR SUMMARY|^ok|Missing|illegal" | sort | uniq -c
