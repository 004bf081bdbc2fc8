"""Run a few batched HMULT+rescale at P-Default for ncu launch lists (development aid)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2212_14191_b200.ckks import CiphertextBatch, CkksContext
from paper_2212_14191_b200.params import CkksParams
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
p = CkksParams.from_preset(sys.argv[2] if len(sys.argv) > 2 else "p_default")
ck = CkksContext(p)
L1, E = p.l_max + 1, p.l_max + 1 + p.k
key = torch.randint(0, 1 << 26, (p.dnum, 2, E, p.n), dtype=torch.int32, device="cuda")
c0 = CiphertextBatch(torch.randint(0, 1 << 26, (2, L1, B, p.n), dtype=torch.int32, device="cuda"), p.l_max)
c1 = CiphertextBatch(torch.randint(0, 1 << 26, (2, L1, B, p.n), dtype=torch.int32, device="cuda"), p.l_max)
fused = len(sys.argv) > 3 and sys.argv[3] == "fused"
op = (lambda: ck.hmult_rescale_batch(c0, c1, key)) if fused else \
    (lambda: ck.rescale_batch(ck.hmult_batch(c0, c1, key)))
for _ in range(2):
    op()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    op()
e.record(); torch.cuda.synchronize()
print(f"{'fused ' if fused else ''}{p.n} B={B}: {s.elapsed_time(e)/3:.2f} ms per hmult+rescale batch -> {3*B/(s.elapsed_time(e)/1e3):.1f}/s")
