"""Per-kernel device times (tfhe_profile_*) of the N=2^16 batched NTT at the
bench shape (45 limbs x B), fwd + inv, several steps."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2212_14191_b200 import _lib, params as par  # noqa: E402
from paper_2212_14191_b200.device import DeviceContext  # noqa: E402
n, L, B = 1 << 16, 45, int(sys.argv[1]) if len(sys.argv) > 1 else 128
primes = par.CkksParams.from_preset("p_default").chain.q
ctx = DeviceContext.get(n, tuple(primes))
x = torch.randint(0, 1 << 28, (L, B, n), dtype=torch.int32, device="cuda")
f, y = torch.empty_like(x), torch.empty_like(x)
for _ in range(3):
    ctx.ntt(x, primes, out=f)
    ctx.ntt(f, primes, inverse=True, out=y)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with _lib.kernel_timer() as kt:
    s.record()
    for _ in range(10):
        ctx.ntt(x, primes, out=f)
        ctx.ntt(f, primes, inverse=True, out=y)
    e.record()
    torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"B={B}: {ms:.3f} ms/step -> {2 * L * B / ms / 1e3:.3f} M limb-NTT/s; " +
      ", ".join(f"{k} {v[1] / v[0]:.3f} ms" for k, v in sorted(kt.times.items())))
