import sys, torch
sys.path.insert(0, ".")
from paper_2212_14191_b200.device import DeviceContext
from paper_2212_14191_b200.params import generate_primes
q0 = generate_primes(1 << 12, [30])
ctx = DeviceContext.get(1 << 12, tuple(q0))
x0 = torch.randint(0, q0[0], (1, 64, 1 << 12), dtype=torch.int64, device="cuda").to(torch.int32)
f0, y0 = torch.empty_like(x0), torch.empty_like(x0)
def cfg0():
    ctx.ntt(x0, q0, out=f0)
    ctx.ntt(f0, q0, inverse=True, out=y0)
for _ in range(3): cfg0()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    cfg0()
y0.zero_()
g.replay(); torch.cuda.synchronize()
print("graph roundtrip exact:", bool(torch.equal(y0, x0)))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("eager", cfg0), ("graph", g.replay)):
    for _ in range(5): fn()
    s.record()
    for _ in range(200): fn()
    e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e) / 200 * 1e3
    print(f"{name}: {us:.1f} us per fwd+inv step -> {2*64/us*1e3:.0f} K limb-NTT/s")
