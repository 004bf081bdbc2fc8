"""Per-kernel device times (tfhe_profile_*) of P-Default HMULT+relin+rescale batches."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2212_14191_b200 import _lib  # noqa: E402
from paper_2212_14191_b200.ckks import CiphertextBatch, CkksContext  # noqa: E402
from paper_2212_14191_b200.params import CkksParams  # noqa: E402
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
p = CkksParams.from_preset(sys.argv[2] if len(sys.argv) > 2 else "p_default")
ck = CkksContext(p)
L1, E = p.l_max + 1, p.l_max + 1 + p.k
key = torch.randint(0, 1 << 26, (p.dnum, 2, E, p.n), dtype=torch.int32, device="cuda")
c0 = CiphertextBatch(torch.randint(0, 1 << 26, (2, L1, B, p.n), dtype=torch.int32, device="cuda"), p.l_max)
c1 = CiphertextBatch(torch.randint(0, 1 << 26, (2, L1, B, p.n), dtype=torch.int32, device="cuda"), p.l_max)
ck.hmult_rescale_batch(c0, c1, key)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with _lib.kernel_timer() as kt:
    s.record()
    for _ in range(2):
        ck.hmult_rescale_batch(c0, c1, key)
    e.record()
    torch.cuda.synchronize()
tot = s.elapsed_time(e) / 2
print(f"B={B}: {tot:.2f} ms per batch -> {B / tot * 1e3:.1f} HMULT/s")
acc = 0.0
for k, (n, ms) in sorted(kt.times.items(), key=lambda kv: -kv[1][1]):
    acc += ms / 2
    print(f"  {k:28s} {n // 2:4d} launches/batch  {ms / 2:8.2f} ms/batch  {100 * ms / 2 / tot:5.1f}%")
print(f"  instrumented kernels {acc:.2f} ms of {tot:.2f}")
