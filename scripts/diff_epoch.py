"""Debug aid: one epoch on the GPU vs the oracle; prints the first mismatching
rows per output with their workflow, its size and the row's position.

  python scripts/diff_epoch.py [c4|c5|c2|swe:N] [--seed S] [--policy srtf] [--flags F]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from nalar_gen import c2, c4, c5, swe_table  # noqa: E402
from oracle import oracle_epoch  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("table", nargs="?", default="c4")
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--policy", default="srtf")
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
if a.table.startswith("swe:"):
    s = swe_table(int(a.table[4:]), a.seed)
else:
    s = {"c2": c2, "c4": c4, "c5": c5}[a.table](a.seed)
o = oracle_epoch(s, a.policy)
ctx = nalar.Context.for_snapshot(s, flags=a.flags)
ctx.upload(s)
ctx.epoch(a.policy)
g = ctx.fetch()
off = s.wf_fut_off.astype(np.int64)
wf = np.repeat(np.arange(s.n_workflows), np.diff(off))
bad = False
for k in ("depth", "status", "level", "instance", "new_pin", "wf_agg", "assign_row"):
    x, y = np.asarray(o[k]), np.asarray(g[k])
    if x.shape != y.shape:
        print(k, "shape", x.shape, y.shape)
        bad = True
        continue
    d = np.nonzero((x != y).reshape(len(x), -1).any(axis=1))[0]
    if len(d):
        bad = True
        print(f"{k}: {len(d)} mismatches")
        for r in d[:12]:
            if k in ("depth", "status", "level", "instance", "new_pin"):
                w = wf[r]
                print(f"   row {r} wf {w} size {off[w + 1] - off[w]} pos {r - off[w]} oracle {x[r]} gpu {y[r]}"
                      f" state {s.f_state[r]}")
            else:
                print(f"   idx {r} oracle {x[r]} gpu {y[r]}")
print("OK" if not bad else "MISMATCH")
