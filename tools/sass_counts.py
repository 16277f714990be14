"""Blackwell-native instruction evidence from the built library (no GPU needed): per decode kernel, the
count of tcgen05 MMAs (UTCHMMA / UTCQMMA), TMEM loads (LDTM), tcgen05 commits (UTCBAR), TMA tensor loads
(UTMALDG), TMA L2 prefetches (UTMAPF/UBLKPF) and mbarrier ops (SYNCS).
usage: python tools/sass_counts.py [paper_2603_11504_b200/liblongflow.so] > profiles/r02_sass_counts.txt"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2603_11504_b200/liblongflow.so"
txt = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ["UTCHMMA", "UTCQMMA", "LDTM", "UTCBAR", "UTMALDG", "UTMAPF", "UBLKPF", "SYNCS", "MUFU.EX2", "SHFL"]
print(f"# cuobjdump -sass {lib}: instruction counts per kernel (static)")
print("kernel".ljust(64) + "".join(k.rjust(10) for k in keys) + "     total")
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n", 1)[0].strip()
    ins = [l for l in f.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,5}\*/", l)]
    short = re.sub(r"_ZN\w*?(tc_decode_kernel|simt_decode_kernel|snapkv\w*?|diag\w*?|deferred_write_kernel|fill_i32)", r"\1", name)[:62]
    cnt = [sum(1 for l in ins if re.search(r"\b" + re.escape(k) + r"\b", l)) for k in keys]
    print(short.ljust(64) + "".join(str(c).rjust(10) for c in cnt) + str(len(ins)).rjust(10))
