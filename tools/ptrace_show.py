"""Print the fused-kernel timeline of CTA 0 from gpurun_out/ptrace_<k>.bin."""
import sys

import numpy as np

N = 128
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(16, N).astype(np.int64)
names = ["P raw", "P a1e", "P done", "MA iss", "MB a2f", "MB iss", "EA acc", "EA a2e", "EA done",
         "EB acc", "EB done", "M accAe"]
t0 = t[t > 0].min()
rel = np.where(t > 0, t - t0, -1)
print("unit " + " ".join(f"{n:>8s}" for n in names))
for u in range(min(int(sys.argv[2]) if len(sys.argv) > 2 else 20, N)):
    if rel[0, u] < 0:
        break
    print(f"{u:4d} " + " ".join(f"{rel[e, u]:8d}" for e in range(len(names))))
d = np.diff(rel[2][rel[2] > 0])
print("producer done-to-done cycles: median", np.median(d) if len(d) else None)
