"""Run the N=2^16 column pass with a TFHE_P3_TRACE build (TFHE_B200_LIB) and
leave the per-unit event clocks of CTA 0 in gpurun_out/ptrace_*.bin."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2212_14191_b200.device import DeviceContext  # noqa: E402
from paper_2212_14191_b200.params import generate_primes  # noqa: E402

n, L, B = 1 << 16, 45, 128
primes = generate_primes(n, [29] * L)
ctx = DeviceContext.get(n, tuple(primes))
x = torch.randint(0, 1 << 28, (L, B, n), dtype=torch.int32, device="cuda")
out = torch.empty_like(x)
for inv in (0, 0):
    ctx.ntt(x, primes, inverse=bool(inv), out=out)
torch.cuda.synchronize()
