"""N = 2^12 timing (development aid): batched fwd / inv NTT (2 limbs x 8192
members, Set_A shape) and Set_A HMULT+relin+rescale; run twice with and
without TFHE_NO_FUSED=1 to A/B the fused single-launch kernel."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2212_14191_b200 import params as par  # noqa: E402
from paper_2212_14191_b200.device import DeviceContext  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


tag = "two-stage" if os.environ.get("TFHE_NO_FUSED") else "fused"
n, L, B = 1 << 12, 2, 8192
primes = par.generate_primes(n, [29] * L)
ctx = DeviceContext.get(n, primes)
x = torch.randint(0, 1 << 28, (L, B, n), dtype=torch.int32, device="cuda")
out = torch.empty_like(x)
for inv in (0, 1):
    ms = timeit(lambda: ctx.ntt(x, primes, inverse=bool(inv), out=out))
    rate = L * B / (ms / 1e3)
    print(f"[{tag}] n=4096 L={L} B={B} inv={inv}: {ms:.3f} ms {rate / 1e6:.1f} M limb-NTT/s "
          f"({8 * n * rate / 1e9:.0f} GB/s compulsory, 8 N B per limb-NTT)", flush=True)
from paper_2212_14191_b200.ckks import CiphertextBatch, CkksContext  # noqa: E402
p = par.CkksParams.from_preset("set_a")
ck = CkksContext(p)
Bh = 4096
L1, E = p.l_max + 1, p.l_max + 1 + p.k
key = torch.randint(0, 1 << 26, (p.dnum, 2, E, p.n), dtype=torch.int32, device="cuda")
c0 = CiphertextBatch(torch.randint(0, 1 << 26, (2, L1, Bh, p.n), dtype=torch.int32, device="cuda"), p.l_max)
c1 = CiphertextBatch(torch.randint(0, 1 << 26, (2, L1, Bh, p.n), dtype=torch.int32, device="cuda"), p.l_max)
ms = timeit(lambda: ck.hmult_rescale_batch(c0, c1, key), 10)
print(f"[{tag}] set_a B={Bh} hmult+relin+rescale: {ms:.3f} ms -> {Bh / (ms / 1e3) / 1e6:.3f} M/s", flush=True)
ms = timeit(lambda: ck.hmult_batch(c0, c1, key), 10)
print(f"[{tag}] set_a B={Bh} hmult+relin: {ms:.3f} ms -> {Bh / (ms / 1e3) / 1e6:.3f} M/s", flush=True)
