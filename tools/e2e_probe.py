"""Probe host<->device copy bandwidth and the host-streaming NTT (development aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2212_14191_b200 import params as par  # noqa: E402
from paper_2212_14191_b200.device import DeviceContext  # noqa: E402

n, L, B = 1 << 16, 45, 128
nbytes = L * B * n * 4
h = torch.empty(nbytes // 4, dtype=torch.int32, pin_memory=True)
d = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms for {nbytes / 2**30:.2f} GiB)")
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2 = h  # noqa
torch.cuda.synchronize()
t = time.perf_counter()
x = torch.empty(nbytes // 4, dtype=torch.int32, pin_memory=True)
print(f"pinned alloc 1st: {(time.perf_counter() - t) * 1e3:.1f} ms")
del x
t = time.perf_counter()
x = torch.empty(nbytes // 4, dtype=torch.int32, pin_memory=True)
print(f"pinned alloc 2nd (cached): {(time.perf_counter() - t) * 1e3:.1f} ms")
primes = par.generate_primes(n, [29] * L)
ctx = DeviceContext.get(n, primes)
xin = h.view(L, B, n)
for i in range(4):
    t = time.perf_counter()
    out = ctx.ntt_host(xin, primes)
    dt = time.perf_counter() - t
    print(f"ntt_host call {i}: {dt * 1e3:.1f} ms -> {L * B / dt / 1e3:.1f} K limb-NTT/s, "
          f"{2 * nbytes / dt / 1e9:.1f} GB/s moved")
    del out
# numpy (pageable) host buffers through batched_apply, as a reference user calls it
import numpy as np  # noqa: E402
from paper_2212_14191_b200.batch import BatchBuffer, batched_apply  # noqa: E402
from paper_2212_14191_b200.ntt import TwiddleTable  # noqa: E402
table = TwiddleTable(n, primes)
table._ctx = ctx
xn = xin.numpy().view(np.uint32).copy()
buf = BatchBuffer(data=xn, basis=primes, domain="coeff")
for i in range(3):
    t = time.perf_counter()
    out = batched_apply(buf, "ntt", table=table)
    dt = time.perf_counter() - t
    print(f"numpy batched_apply ntt {i}: {dt * 1e3:.1f} ms -> {L * B / dt / 1e3:.1f} K limb-NTT/s")
