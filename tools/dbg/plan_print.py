import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from bench import workload_of
from paper_2603_11504_b200 import Cache
for w in sys.argv[1:]:
    wl = workload_of(w)
    c = Cache(wl.B, wl.Hq, wl.Hkv, wl.d, wl.N, out_dtype="bf16")
    print(os.environ.get("LF_LIB", "default"), w, c.plan())
