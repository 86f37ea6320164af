"""Run a few policy epochs on one table, for ncu (no timing printed here).

  python scripts/profile_epoch.py [--n 131072] [--epochs 5] [--policy srtf] [--flags 0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from nalar_gen import swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 17)
ap.add_argument("--epochs", type=int, default=5)
ap.add_argument("--policy", default="srtf")
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
s = swe_table(a.n, seed=a.seed)
ctx = nalar.Context.for_snapshot(s, flags=a.flags)
ctx.upload(s)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.ExternalStream(ctx.stream)
for _ in range(a.epochs):
    with torch.cuda.stream(stream):
        flush.zero_()
    ctx.epoch(a.policy)
torch.cuda.synchronize()
st = ctx.stats()
print("n", s.n_futures, "ready", st.n_ready, "eligible", st.n_eligible, "assigned", st.n_assigned)
