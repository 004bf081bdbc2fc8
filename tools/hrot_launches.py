"""A few P-Default HROTATE batches (ncu launch-list aid)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2212_14191_b200.ckks import CiphertextBatch, CkksContext  # noqa: E402
from paper_2212_14191_b200.params import CkksParams  # noqa: E402
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
p = CkksParams.from_preset("p_default")
ck = CkksContext(p)
L1, E = p.l_max + 1, p.l_max + 1 + p.k
key = torch.randint(0, 1 << 26, (p.dnum, 2, E, p.n), dtype=torch.int32, device="cuda")
c0 = CiphertextBatch(torch.randint(0, 1 << 26, (2, L1, B, p.n), dtype=torch.int32, device="cuda"), p.l_max)
for _ in range(3):
    ck.hrotate_batch(c0, 1, key)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    ck.hrotate_batch(c0, 1, key)
e.record()
torch.cuda.synchronize()
print(f"HROTATE B={B}: {s.elapsed_time(e) / 3:.2f} ms per batch -> {3 * B / (s.elapsed_time(e) / 1e3):.1f}/s")
