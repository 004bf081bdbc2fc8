"""N = 2^16 batched NTT timing (development aid): fwd / inv over the 45
p_default primes x B members; TFHE_NO_P3=1 times the 256 x 256 TS plan."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2212_14191_b200.device import DeviceContext  # noqa: E402
from paper_2212_14191_b200.params import CkksParams  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


tag = "ts" if os.environ.get("TFHE_NO_P3") else "p3"
p = CkksParams.from_preset("p_default")
primes = list(p.chain.q)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = DeviceContext.get(1 << 16, tuple(primes))
L = len(primes)
q = torch.tensor(primes, dtype=torch.int64, device="cuda").view(L, 1, 1)
x = (torch.randint(0, 1 << 62, (L, B, 1 << 16), device="cuda") % q).to(torch.int32)
out = torch.empty_like(x)
for inv in (0, 1):
    ms = timeit(lambda: ctx.ntt(x, primes, inverse=bool(inv), out=out))
    rate = L * B / (ms / 1e3)
    print(f"[{tag}] N=2^16 L={L} B={B} inv={inv}: {ms:.3f} ms  {rate / 1e6:.3f} M limb-NTT/s "
          f"({8 * 65536 * rate / 1e9:.0f} GB/s compulsory)", flush=True)
