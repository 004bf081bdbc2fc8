"""Summarise a TFHE_TS_TRACE dump (per-chunk clock64 events of CTA 0)."""
import sys
import numpy as np
for fn in sys.argv[1:]:
    t = np.fromfile(fn, dtype=np.uint64).reshape(16, 512).astype(np.int64)
    n = int((t[5] > 0).sum())
    t0 = t[5][0]
    T = lambda e: np.where(t[e][:n] > 0, t[e][:n] - t0, -1)
    lo = 100
    print(fn, "chunks", n)
    ev2 = T(2)[lo:n]
    iss = (T(2) - T(1))[lo:n]; wt = (T(1) - T(0))[lo:n]
    print("  MMA issue", iss[iss > 0].mean(), " wait", wt[wt >= 0].mean(), " issue-end period", np.diff(ev2).mean())
    print("  epi w4: wait", (T(5) - T(4))[lo:n].mean(), " ld", (T(6) - T(5))[lo:n].mean(),
          " period", np.diff(T(5)[lo:n]).mean())
    if (t[15] > 0).sum():
        print("  epi w4 after-ld -> combined", (T(15) - T(6))[lo:n].mean(), " -> store end", (T(13) - T(15))[lo:n].mean(),
              " store end -> next wait", (T(4)[lo+1:n] - T(13)[lo:n-1]).mean())
    print("  prod: raw wait", (T(8) - T(7))[lo:n].mean(), " b_empty wait", (T(9) - T(8))[lo:n].mean(),
          " convert", (T(10) - T(9))[lo:n].mean(), " period", np.diff(T(10)[lo:n]).mean())
