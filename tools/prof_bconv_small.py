"""Time the element-wise base conversion (K=2 specials -> 2 chain rows, Set_A ModDown shape)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2212_14191_b200.ckks import CkksContext  # noqa: E402
from paper_2212_14191_b200.params import CkksParams  # noqa: E402
p = CkksParams.from_preset("set_a")
ck = CkksContext(p)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
src = torch.randint(0, 1 << 26, (len(p.chain.p), B, p.n), dtype=torch.int32, device="cuda")
dst = torch.empty((len(p.chain.q), B, p.n), dtype=torch.int32, device="cuda")
for _ in range(3):
    ck.dev.bconv(src, p.chain.p, p.chain.q, out=dst)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    ck.dev.bconv(src, p.chain.p, p.chain.q, out=dst)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
nb = 4 * (len(p.chain.p) + len(p.chain.q)) * B * p.n
print(f"bconv_small {len(p.chain.p)}->{len(p.chain.q)} B={B}: {ms:.3f} ms, {nb / ms / 1e6:.0f} GB/s")
