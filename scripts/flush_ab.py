"""Epoch time with and without the L2 flush between epochs (C1 / C2 / C4):
how much of the epoch is cold-cache latency (data and instructions)?
  python scripts/flush_ab.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import c1, c2, c4  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
small = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
res = {}
for name, s in (("c1", c1()), ("c2", c2(1)), ("c4", c4())):
    ctx = nalar.Context.for_snapshot(s)
    ctx.upload(s)
    st = torch.cuda.ExternalStream(ctx.stream)
    for mode in ("flush", "warm", "flush64"):
        ts = []
        for i in range(210):
            if mode == "flush":
                flush.zero_()
            elif mode == "flush64":
                small.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            ctx.epoch("srtf")
            b.record(st)
            torch.cuda.synchronize()
            if i >= 10:
                ts.append(a.elapsed_time(b) * 1e3)
        res[f"{name}_{mode}"] = round(float(np.mean(ts)), 2)
    ctx.close()
print(json.dumps(res))
