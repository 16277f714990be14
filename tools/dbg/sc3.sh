S=/usr/local/cuda/bin/compute-sanitizer
echo "== synccheck S=8 k=2 B=40"; timeout 600 $S --tool synccheck --print-limit 6 python tools/dbg/one_step.py 40 28 4 1011 128 2 2 3 2>&1 | grep -v "Host Frame" | head -60
echo "== synccheck S=8 k=2 B=40 lat off"; timeout 600 $S --tool synccheck --print-limit 3 python tools/dbg/one_step.py 40 28 4 1011 128 2 1 3 2>&1 | grep -v "Host Frame" | head -30
echo "== synccheck S=8 k=1 B=40"; timeout 600 $S --tool synccheck --print-limit 3 python tools/dbg/one_step.py 40 28 4 1011 128 1 2 3 2>&1 | grep -v "Host Frame" | head -20
echo "== synccheck S=4 k=2 B=40"; timeout 600 $S --tool synccheck --print-limit 3 python tools/dbg/one_step.py 40 28 4 500 128 2 2 3 2>&1 | grep -v "Host Frame" | head -20
