"""A few epochs of a one-workflow SWE table (the plain K1 build): a clean
single-block target for ncu.   python scripts/solo_epoch.py [--n 190] [--seed 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from nalar_gen import swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=190)
ap.add_argument("--seed", type=int, default=3)
ap.add_argument("--epochs", type=int, default=3)
a = ap.parse_args()
s = swe_table(a.n, a.seed, p_deep=0.0)
ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_NO_GRAPH)
ctx.upload(s)
for _ in range(a.epochs):
    ctx.epoch("srtf")
torch.cuda.synchronize()
print("ok", s.n_futures, s.n_workflows)
