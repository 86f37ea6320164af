"""What can a 2.3 MB pinned H2D / 0.4 MB D2H move per call on this box?
DMA (cudaMemcpyAsync via torch) at a few sizes, for the e2e upload/fetch budget."""
import json
import time

import torch

res = {}
for mb in (0.4, 1.0, 2.3, 8.0):
    n = int(mb * 1e6)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for direction in ("h2d", "d2h"):
        ts = []
        for i in range(30):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if direction == "h2d":
                d.copy_(h, non_blocking=True)
            else:
                h.copy_(d, non_blocking=True)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        ts.sort()
        res[f"{direction}_{mb}MB_us_p50"] = round(ts[len(ts) // 2] * 1e6, 1)
        res[f"{direction}_{mb}MB_GBps"] = round(n / ts[len(ts) // 2] / 1e9, 1)
# the empty sync round trip
ts = []
for i in range(30):
    t0 = time.perf_counter(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
res["sync_us"] = round(sorted(ts)[15] * 1e6, 1)
print(json.dumps(res, indent=1))
