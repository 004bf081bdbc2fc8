"""Run the HBM-bound kernels once each at the bench shape (ncu aid):
hada_mult, ele_add, NTT-domain automorphism, HMULT tensor product."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2212_14191_b200 import _lib  # noqa: E402
from paper_2212_14191_b200.device import DeviceContext, _ptr, _stream  # noqa: E402
from paper_2212_14191_b200.params import CkksParams  # noqa: E402
p = CkksParams.from_preset("p_default")
primes = list(p.chain.q)
L, B, N = len(primes), 128, p.n
ctx = DeviceContext.get(N, tuple(p.chain.q) + tuple(p.chain.p), n_chain=L, n_special=1)
x = torch.randint(0, 1 << 28, (L, B, N), dtype=torch.int32, device="cuda")
y = torch.randint(0, 1 << 28, (L, B, N), dtype=torch.int32, device="cuda")
o = torch.empty_like(x)
for _ in range(2):
    ctx.eltwise(_lib.OP_MUL, x, y, primes, out=o)
    ctx.eltwise(_lib.OP_ADD, x, y, primes, out=o)
    ctx.automorphism(x, 5, True, primes, out=o)
    ct0 = x.view(L, 2, B // 2, N).transpose(0, 1).contiguous()
    ct1 = y.view(L, 2, B // 2, N).transpose(0, 1).contiguous()
    tp = torch.empty((3, L, B // 2, N), dtype=torch.int32, device="cuda")
    _lib.check(ctx.lib.tfhe_tensor_product(ctx.handle, _ptr(ct0), _ptr(ct1), 0, L, B // 2,
                                           _ptr(tp), _stream(ctx.device)), "tensor")
    del ct0, ct1, tp
torch.cuda.synchronize()
