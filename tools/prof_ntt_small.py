"""Batched NTT at N=2^12 (Set_A-like: 2 limbs x B) for ncu (development aid)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2212_14191_b200 import params as par  # noqa: E402
from paper_2212_14191_b200.device import DeviceContext  # noqa: E402
n, L = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 12, 2
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
primes = par.generate_primes(n, [29] * L)
ctx = DeviceContext.get(n, primes)
x = torch.randint(0, 1 << 28, (L, B, n), dtype=torch.int32, device="cuda")
out = torch.empty_like(x)
for _ in range(3):
    ctx.ntt(x, primes, out=out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    ctx.ntt(x, primes, out=out)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"n={n} L={L} B={B}: {ms:.3f} ms -> {L * B / ms / 1e3:.2f} M limb-NTT/s, "
      f"{L * B * n * 8 / ms / 1e6:.0f} GB/s compulsory")
