"""Raw concurrent H2D + D2H bandwidth over pinned buffers (the e2e ceiling; development aid)."""
import time
import torch

nb = 1 << 30
ha = torch.empty(nb // 4, dtype=torch.int32, pin_memory=True)
hb = torch.empty(nb // 4, dtype=torch.int32, pin_memory=True)
da = torch.empty(nb // 4, dtype=torch.int32, device="cuda")
db = torch.empty(nb // 4, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for chunk in (1 << 22, 1 << 24, 1 << 26, nb):
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for off in range(0, nb // 4, chunk // 4):
            with torch.cuda.stream(s1):
                da[off:off + chunk // 4].copy_(ha[off:off + chunk // 4], non_blocking=True)
            with torch.cuda.stream(s2):
                hb[off:off + chunk // 4].copy_(db[off:off + chunk // 4], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"duplex chunk {chunk >> 20} MiB: {2 * nb / dt / 1e9:.1f} GB/s total ({nb / dt / 1e9:.1f} each way)")
