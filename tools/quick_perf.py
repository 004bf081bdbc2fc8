"""Quick device timing of the NTT and CKKS ops (development aid, not the bench)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2212_14191_b200 import params as par  # noqa: E402
from paper_2212_14191_b200.device import DeviceContext  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def ntt_perf(n, L, B):
    primes = par.generate_primes(n, [29] * L)
    ctx = DeviceContext.get(n, primes)
    x = torch.randint(0, 1 << 28, (L, B, n), dtype=torch.int32, device="cuda")
    out = torch.empty_like(x)
    for inv in (0, 1):
        ms = timeit(lambda: ctx.ntt(x, primes, inverse=bool(inv), out=out))
        rate = L * B / (ms / 1e3)
        print(f"n={n} L={L} B={B} inv={inv}: {ms:.3f} ms  {rate/1e6:.3f} M limb-NTT/s "
              f"({rate/L/1e3:.1f} K poly-NTT/s)", flush=True)


def ckks_perf(preset, B):
    from paper_2212_14191_b200.ckks import CkksContext, CiphertextBatch
    p = par.CkksParams.from_preset(preset)
    ctx = CkksContext(p)
    L1 = p.l_max + 1
    E = L1 + p.k
    key = torch.randint(0, 1 << 26, (p.dnum, 2, E, p.n), dtype=torch.int32, device="cuda")
    ct0 = CiphertextBatch(torch.randint(0, 1 << 26, (2, L1, B, p.n), dtype=torch.int32,
                                        device="cuda"), p.l_max)
    ct1 = CiphertextBatch(torch.randint(0, 1 << 26, (2, L1, B, p.n), dtype=torch.int32,
                                        device="cuda"), p.l_max)
    ms = timeit(lambda: ctx.hmult_batch(ct0, ct1, key), reps=3)
    print(f"{preset} B={B} hmult: {ms:.2f} ms -> {B/(ms/1e3):.1f} HMULT/s", flush=True)
    ms = timeit(lambda: ctx.rescale_batch(ct0), reps=3)
    print(f"{preset} B={B} rescale: {ms:.2f} ms -> {B/(ms/1e3):.1f} /s", flush=True)
    ms = timeit(lambda: ctx.hrotate_batch(ct0, 1, key), reps=3)
    print(f"{preset} B={B} hrotate: {ms:.2f} ms -> {B/(ms/1e3):.1f} /s", flush=True)


if __name__ == "__main__":
    ntt_perf(1 << 16, 45, 128)
    ntt_perf(1 << 12, 2, 8192)
    ntt_perf(1 << 12, 1, 64)
    ckks_perf("set_a", 4096)
    ckks_perf("p_default", 32)
