"""Histogram of C4 epoch times (graph replay, L2 flushed before each, CUDA
events tick in 0.512 us) and the run structure of slow epochs.
  python scripts/epoch_hist.py [--n 2000]"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2000)
ap.add_argument("--flush", type=int, default=1)
a = ap.parse_args()
s = swe_table(1 << 17, 1)
ctx = nalar.Context.for_snapshot(s)
ctx.upload(s)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.ExternalStream(ctx.stream)
ev = []
with torch.cuda.stream(st):
    for i in range(a.n + 20):
        if a.flush:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.epoch("srtf")
        e1.record(st)
        ev.append((e0, e1))
torch.cuda.synchronize()
t = np.array([x.elapsed_time(y) * 1e3 for x, y in ev[20:]])
c = collections.Counter(np.round(t, 2))
print("mean", t.mean().round(2), "p50", np.median(t).round(2))
for k in sorted(c):
    print(f"  {k:7.2f} us  {c[k]:5d}")
slow = t > np.median(t) + 1.0
runs = np.diff(np.flatnonzero(np.diff(np.r_[0, slow.astype(int), 0])))
print("slow fraction", slow.mean().round(3), "first 40 flags", "".join("x" if v else "." for v in slow[:40]))
