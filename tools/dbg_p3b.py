import os, sys, numpy as np, torch
os.environ["TFHE_P3_DBG"]="1"
sys.path.insert(0,'.')
from oracle import oracle as O
from paper_2212_14191_b200.device import DeviceContext
from paper_2212_14191_b200.params import generate_primes
n=1<<16
L,B=1,300
primes=generate_primes(n,[29])
q=primes[0]
ctx=DeviceContext.get(n,tuple(primes))
rng=np.random.default_rng(7)
x=O.uniform_rows(rng,primes,(B,n))
PT=ctx.ntt(torch.from_numpy(x.view(np.int32)).cuda(),primes).cpu().numpy().view(np.uint32).reshape(B,64,1024)
psi=O.negacyclic_root(q,n)
k1=np.arange(1024,dtype=np.uint64)
bad=0
for b in range(0,B,7):
    A=x[0,b].reshape(1024,64)           # A[i1][i2]
    S=O.ntt(np.ascontiguousarray(A.T)[None],[q])[0]   # S[i2][k1] = 1024-point negacyclic NTT of column i2
    for i2 in range(64):
        h=np.array([pow(psi,((2*int(kk)+1)*i2)%(2*n),q) for kk in range(1024)],dtype=np.uint64)
        want=(S[i2].astype(np.uint64)*h % q)
        got=PT[b,i2].astype(np.uint64) % q
        d=np.nonzero(got!=want)[0]
        if len(d):
            bad+=1
            if bad<12: print("member",b,"i2",i2,"bad k1",d[:8].tolist(),"n",len(d), "b2set",sorted(set((d//32).tolist()))[:10], "b1set", sorted(set((d%32).tolist()))[:10])
print("bad (member,i2) pairs", bad)
