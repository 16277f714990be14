import numpy as np, sys
a = np.load(sys.argv[1]).astype(np.float64)
used = a[:, 0, 6] > 0
for c in np.nonzero(used)[0][:2]:
    t0 = a[c, 0, 16]
    k = a[c, 32, :32]; v = a[c, 33, :32]
    print("cta", c, "entry->start %.2f maxdone %.2f Vdone %.2f r0done %.2f" % tuple((a[c, 0, j] - t0) / 1e3 for j in (0, 1, 2, 14)))
    iss = a[c, 34, :32]
    print("  tiles issued (us):  ", " ".join("%.1f" % ((x - t0) / 1e3) for x in iss if x > 0))
    print("  K tiles landed (us):", " ".join("%.1f" % ((x - t0) / 1e3) for x in k if x > 0))
    print("  V P-ready (us):     ", " ".join("%.1f" % ((x - t0) / 1e3) for x in v if x > 0))
