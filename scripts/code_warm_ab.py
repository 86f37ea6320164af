"""How much of a cold (L2-flushed) epoch is instruction fetch?  Epoch of table A
timed after (a) the flush only, (b) the flush and then an epoch of ANOTHER
context (table B: same kernels, disjoint data -- warms the code, not A's
data), (c) no flush.
  python scripts/code_warm_ab.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import c1, c2, swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
pairs = (("c1", c1(), c2(2)), ("c2", c2(1), c2(2)), ("c4", swe_table(1 << 17, 1), swe_table(1 << 17, 2)))
for name, sa, sb in pairs:
    ca = nalar.Context.for_snapshot(sa)
    ca.upload(sa)
    cb = nalar.Context.for_snapshot(sb)
    cb.upload(sb)
    st = torch.cuda.ExternalStream(ca.stream)
    for mode in ("flush", "flush_codewarm", "warm"):
        ts = []
        for i in range(160):
            if mode != "warm":
                flush.zero_()
                torch.cuda.synchronize()
            if mode == "flush_codewarm":
                cb.epoch("srtf")
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            ca.epoch("srtf")
            b.record(st)
            torch.cuda.synchronize()
            if i >= 10:
                ts.append(a.elapsed_time(b) * 1e3)
        res[f"{name}_{mode}"] = round(float(np.median(ts)), 2)
    ca.close()
    cb.close()
    print(name, {k: v for k, v in res.items() if k.startswith(name)}, flush=True)
print(json.dumps(res))
