"""Where does the end-to-end (public API) step go?  Times upload / epoch /
fetch separately (wall clock, pinned host buffers, C4 table).

  python scripts/e2e_breakdown.py [--steps 50]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import Snapshot, c4  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
a = ap.parse_args()
s = c4()
keep = []


def pinned_like(x):
    t = torch.empty(max(x.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    keep.append(t)
    v = t.numpy()[:x.nbytes].view(x.dtype).reshape(x.shape)
    v[...] = x
    return v


sp = Snapshot(global_row_base=s.global_row_base, name=s.name, **{k: pinned_like(v) for k, v in s.arrays().items()})
ctx = nalar.Context.for_snapshot(sp)
ctx.upload(sp)
outb = ctx.output_buffers(("status", "instance", "assign"), alloc=lambda n, dt: pinned_like(np.zeros(n, dt)))
T = {"upload": [], "epoch_sync": [], "fetch": [], "total": []}
for i in range(5 + a.steps):
    t0 = time.perf_counter()
    ctx.upload(sp)
    t1 = time.perf_counter()
    ctx.epoch("srtf")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ctx.fetch(("status", "instance", "assign"), out=outb)
    t3 = time.perf_counter()
    if i >= 5:
        T["upload"].append(t1 - t0); T["epoch_sync"].append(t2 - t1); T["fetch"].append(t3 - t2)
        T["total"].append(t3 - t0)
res = {k: float(np.median(v) * 1e6) for k, v in T.items()}
# pieces of upload
tt = []
for i in range(20):
    t0 = time.perf_counter()
    nalar.snapshot_struct(sp)
    tt.append(time.perf_counter() - t0)
res["snapshot_struct_marshal_us"] = float(np.median(tt) * 1e6)
print(json.dumps(res, indent=1))
