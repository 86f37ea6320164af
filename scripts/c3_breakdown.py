"""C3 (dynamic, 80 RPS) per-epoch breakdown: epoch, fetch, delta apply (wall clock).

  python scripts/c3_breakdown.py [--epochs 60]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import RouterSim  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--epochs", type=int, default=60)
a = ap.parse_args()
sim = RouterSim(1)
sim.warmup(450)
s = sim.snapshot()
ctx = nalar.Context(200000, 400000, 20000, 32, 4)
ctx.upload(s)
keep = []


def pinned(n, dt):
    t = torch.empty(max(n * np.dtype(dt).itemsize, 1), dtype=torch.uint8, pin_memory=True)
    keep.append(t)
    return t.numpy()[:n * np.dtype(dt).itemsize].view(dt)


outb = {"new_pin": pinned(200000, np.uint8), "assign_row": pinned(200000, np.uint32),
        "assign_inst": pinned(200000, np.int16)}
T = {"epoch": [], "fetch": [], "delta": [], "sim": []}
for k in range(a.epochs):
    t0 = time.perf_counter()
    ctx.epoch("srtf")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = ctx.fetch(("new_pin", "assign"), out=outb)
    r["new_pin"] = r["new_pin"][:ctx.n[0]]
    t2 = time.perf_counter()
    d = sim.step(r["assign_row"], r["assign_inst"], r["new_pin"])
    t3 = time.perf_counter()
    t3b = time.perf_counter()
    nalar.delta_struct(d)
    t3c = time.perf_counter()
    T.setdefault("marshal", []).append(t3c - t3b)
    t3 = time.perf_counter()
    ctx.apply_delta(d)
    t4 = time.perf_counter()
    T["epoch"].append(t1 - t0); T["fetch"].append(t2 - t1); T["sim"].append(t3 - t2); T["delta"].append(t4 - t3)
print(json.dumps({k + "_us_p50": float(np.median(v) * 1e6) for k, v in T.items()}, indent=1))
