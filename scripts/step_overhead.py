"""nalar_step at C4 (pinned in / out): the Python binding's share of the call
(ctx.step vs the bare ctypes call on the same marshalled structs).
  python scripts/step_overhead.py"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import Snapshot, c4  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

s = c4()
keep = []


def pinned_like(x):
    t = torch.empty(max(x.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    keep.append(t)
    v = t.numpy()[:x.nbytes].view(x.dtype).reshape(x.shape)
    v[...] = x
    return v


sp = Snapshot(global_row_base=0, name=s.name, **{k: pinned_like(v) for k, v in s.arrays().items()})
ctx = nalar.Context.for_snapshot(s)
F = ("status", "level", "instance", "new_pin", "assign")
out = ctx.output_buffers(F, alloc=lambda n, dt: pinned_like(np.zeros(n, dt)), like=s)
for _ in range(20):
    ctx.step(sp, "srtf", F, out=out)
st = ctx._snap(sp)
d = ctx._decisions(out, True)
row = C.c_int64(-1)
lib = nalar._lib
a, b, parts = [], [], {"snap": [], "dec": [], "res": []}
for i in range(300):
    t0 = time.perf_counter()
    ctx.step(sp, "srtf", F, out=out)
    t1 = time.perf_counter()
    lib.nalar_step(ctx.h, C.byref(st), 1, C.byref(d), C.byref(row))
    t2 = time.perf_counter()
    x0 = time.perf_counter(); ctx._snap(sp); x1 = time.perf_counter(); ctx._decisions(out, True)
    x2 = time.perf_counter(); ctx._results(out, d); x3 = time.perf_counter()
    a.append(t1 - t0); b.append(t2 - t1)
    parts["snap"].append(x1 - x0); parts["dec"].append(x2 - x1); parts["res"].append(x3 - x2)
print(json.dumps({"ctx_step_us": float(np.median(a) * 1e6), "bare_c_us": float(np.median(b) * 1e6),
                  **{k + "_us": float(np.median(v) * 1e6) for k, v in parts.items()}}))
