"""Run the alpha=9 -> 54-target tensor-core base conversion a few times (ncu aid)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2212_14191_b200.ckks import CkksContext  # noqa: E402
from paper_2212_14191_b200.params import CkksParams  # noqa: E402
pd = CkksParams.from_preset("p_dnum5")
ck = CkksContext(pd)
ext = tuple(pd.chain.q) + tuple(pd.chain.p)
B, N = int(sys.argv[1]) if len(sys.argv) > 1 else 32, pd.n
src = torch.randint(0, 1 << 28, (pd.alpha, B, N), dtype=torch.int32, device="cuda")
dst = torch.empty((len(ext), B, N), dtype=torch.int32, device="cuda")
for _ in range(3):
    ck.dev.bconv(src, pd.chain.q[:pd.alpha], ext, out=dst)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    ck.dev.bconv(src, pd.chain.q[:pd.alpha], ext, out=dst)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"bconv {pd.alpha}->{len(ext)} B={B}: {ms:.3f} ms, {4 * (pd.alpha + len(ext)) * B * N / ms / 1e6:.0f} GB/s")
