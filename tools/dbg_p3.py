"""Reproducer of the raw-slot reuse race in the N=2^16 passes (multi-unit CTAs): fixed by the
fence.proxy.async before a TMA-filled slot is released; kept as a regression aid."""
import sys, numpy as np, torch
sys.path.insert(0,'.')
from oracle import oracle as O
from paper_2212_14191_b200.device import DeviceContext
from paper_2212_14191_b200.params import generate_primes
n=1<<16
for (L,B) in [(1,1),(1,2),(1,8),(1,37),(2,37),(5,4),(5,37),(1,300)]:
    primes=generate_primes(n,[29,31,30,28,26][:L])
    ctx=DeviceContext.get(n,tuple(primes))
    rng=np.random.default_rng(L*100+B)
    x=O.uniform_rows(rng,primes,(B,n))
    f=ctx.ntt(torch.from_numpy(x.view(np.int32)).cuda(),primes).cpu().numpy().view(np.uint32)
    w=O.ntt(x,primes)
    bad=np.argwhere((f!=w).any(axis=2))
    print(L,B,"bad rows",len(bad), bad[:10].tolist(), flush=True)
    if len(bad):
        l,b=bad[0]; d=np.nonzero(f[l,b]!=w[l,b])[0]
        print("  first bad positions", d[:20].tolist(), "count", len(d))
        print("  k1 set", sorted(set((d%1024).tolist()))[:20], "k2 set", sorted(set((d//1024).tolist()))[:20])
    fi=ctx.ntt(torch.from_numpy(w.view(np.int32)).cuda(),primes,inverse=True).cpu().numpy().view(np.uint32)
    print("  inverse roundtrip ok", np.array_equal(fi,x))
