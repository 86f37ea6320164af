"""Per-workflow K1 P2 durations (NALAR_F_PROFILE stamps): how long does a
workflow's sweep take as a function of its rows, long / short, wide rows?

  python scripts/wf_times.py [--n 131072] [--seed 1] [--table c4|c2|c1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import c1, c2, swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 17)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--table", default="c4")
a = ap.parse_args()
s = {"c4": lambda: swe_table(a.n, a.seed), "c2": lambda: c2(a.seed), "c1": c1}[a.table]()
ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_PROFILE | nalar.NALAR_F_NO_GRAPH)
ctx.upload(s)
for _ in range(3):
    ctx.epoch("srtf")
torch.cuda.synchronize()
pr = nalar.nalar_debug_profile(ctx.h).astype(np.int64)
W, R = s.n_workflows, s.n_instances + s.n_types
B = (len(pr) - 2 * W - 8 * R - 4 * W) // 16
wf = pr[:2 * W].reshape(W, 2)
blk = pr[2 * W:2 * W + 8 * B].reshape(B, 8)
t0 = blk[:, 3].min()
off = s.wf_fut_off.astype(np.int64)
rows = np.diff(off)
eoff = s.f_edge_off.astype(np.int64)
wide = np.array([(np.diff(eoff[off[w]:off[w + 1] + 1]) > 4).sum() for w in range(W)])
dur = (wf[:, 1] - wf[:, 0]) / 1e3
start = (wf[:, 0] - t0) / 1e3
end = (wf[:, 1] - t0) / 1e3
lng = rows >= 128
for name, m in (("short", ~lng), ("long", lng)):
    if not m.any():
        continue
    print(f"{name}: n={m.sum()} rows mean {rows[m].mean():.0f}  dur us p50 {np.median(dur[m]):.2f} max {dur[m].max():.2f}"
          f"  start p50 {np.median(start[m]):.2f} max {start[m].max():.2f}  end max {end[m].max():.2f}"
          f"  ns/row {1e3 * dur[m].sum() / rows[m].sum():.1f}  wide rows/wf {wide[m].mean():.2f}")
order = np.argsort(-end)[:8]
for w in order:
    print(f"  wf {w} rows {rows[w]} wide {wide[w]} start {start[w]:.2f} dur {dur[w]:.2f} end {end[w]:.2f}")
# blocks: staged time, p2 end
tx = pr[2 * W + 8 * B + 8 * R + 4 * W:2 * W + 8 * B + 8 * R + 4 * W + 8 * B].reshape(B, 8)
n = max(tx[:, 3].sum(), 1)
print(f"warp steps {tx[:, 3].sum()}: cycles/step load {tx[:, 0].sum() / n:.0f} settle {tx[:, 1].sum() / n:.0f} "
      f"store {tx[:, 2].sum() / n:.0f}  rounds/step {tx[:, 4].sum() / n:.1f}  wide steps {tx[:, 5].sum()}")
print("pre-pass end us p50", np.median((blk[:, 6] - t0) / 1e3))
print("block staged us p50", np.median((blk[:, 0] - t0) / 1e3), "p2 end p50", np.median((blk[:, 7] - t0) / 1e3))
