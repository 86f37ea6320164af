"""C5 (2^20 futures) epoch on one GPU, L2 flushed, under the current
environment: mean / p50 epoch us and K1 blocks.  python scripts/c5_ab.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import c5  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

s = c5(1)
ctx = nalar.Context.for_snapshot(s)
ctx.upload(s)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.ExternalStream(ctx.stream)
ts = []
for i in range(60):
    flush.zero_()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    ctx.epoch("srtf")
    b.record(st)
    torch.cuda.synchronize()
    if i >= 10:
        ts.append(a.elapsed_time(b) * 1e3)
print(json.dumps({"env_x2": os.environ.get("NALAR_K1_X2"), "epoch_us_mean": float(np.mean(ts)),
                  "p50": float(np.median(ts))}))
