"""Set_A HMULT+rescale with a TFHE_FUSED_TRACE build: one ftrace_<k>.bin per fused launch."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2212_14191_b200.ckks import CiphertextBatch, CkksContext  # noqa: E402
from paper_2212_14191_b200.params import CkksParams  # noqa: E402
p = CkksParams.from_preset("set_a")
ck = CkksContext(p)
B = 4096
L1, E = p.l_max + 1, p.l_max + 1 + p.k
key = torch.randint(0, 1 << 26, (p.dnum, 2, E, p.n), dtype=torch.int32, device="cuda")
c0 = CiphertextBatch(torch.randint(0, 1 << 25, (2, L1, B, p.n), dtype=torch.int32, device="cuda"), p.l_max)
c1 = CiphertextBatch(torch.randint(0, 1 << 25, (2, L1, B, p.n), dtype=torch.int32, device="cuda"), p.l_max)
ck.hmult_rescale_batch(c0, c1, key)
torch.cuda.synchronize()
