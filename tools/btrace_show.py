"""Print the bconv_tc timeline of CTA 0 from gpurun_out/btrace_<k>.bin (TFHE_BC_TRACE build)."""
import sys

import numpy as np

N = 128
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(16, N).astype(np.int64)
names = ["P a_emp", "P raw", "P a_full", "M a_full", "M acc0e", "M acc1e", "E0 accf", "E0 rel",
         "E0 done", "E1 accf", "E1 rel", "E1 done", "P refill", "E0 copy", "E1 copy", "E bar"]
t0 = t[t > 0].min()
rel = np.where(t > 0, t - t0, -1)
print("tile " + " ".join(f"{n:>8s}" for n in names))
for u in range(min(int(sys.argv[2]) if len(sys.argv) > 2 else 24, N)):
    if rel[0, u] < 0:
        break
    print(f"{u:4d} " + " ".join(f"{rel[e, u]:8d}" for e in range(len(names))))
for e, nm in ((2, "producer a_full"), (3, "MMA a_full"), (8, "E0 done"), (11, "E1 done")):
    d = np.diff(rel[e][rel[e] > 0])
    print(f"{nm} step cycles: median {np.median(d) if len(d) else None}")
