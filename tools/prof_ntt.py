"""Run a few N=2^16 batched NTTs for ncu capture (development aid)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2212_14191_b200 import params as par
from paper_2212_14191_b200.device import DeviceContext
n, L, B = 1 << 16, 45, int(sys.argv[1]) if len(sys.argv) > 1 else 128
primes = par.generate_primes(n, [29] * L)
ctx = DeviceContext.get(n, primes)
x = torch.randint(0, 1 << 28, (L, B, n), dtype=torch.int32, device="cuda")
out = torch.empty_like(x)
back = torch.empty_like(x)
for _ in range(2):
    ctx.ntt(x, primes, out=out)
    ctx.ntt(out, primes, inverse=True, out=back)
torch.cuda.synchronize()
