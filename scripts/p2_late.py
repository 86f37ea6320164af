"""The latest-ending workflows of K1's P2 at C4 (NALAR_F_PROFILE stamps):
rows, depth, start / end (us from kernel entry), compose wait cycles, and the
per-block transfer phase cycle sums.
  python scripts/p2_late.py [--seed 1] [--deep 0.05]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--deep", type=float, default=0.05)
ap.add_argument("--flush", type=int, default=1)
a = ap.parse_args()
s = swe_table(1 << 17, a.seed, p_deep=a.deep)
ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_PROFILE | nalar.NALAR_F_NO_GRAPH)
ctx.upload(s)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(4):
    if a.flush:
        with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream)):
            flush.zero_()
    ctx.epoch("srtf")
torch.cuda.synchronize()
pr = nalar.nalar_debug_profile(ctx.h).astype(np.int64)
W, R = s.n_workflows, s.n_instances + s.n_types
B = (len(pr) - 2 * W - 8 * R - 4 * W) // 16
o1, o2 = 2 * W, 2 * W + 8 * B
o3, o4 = o2 + 8 * R, o2 + 8 * R + 4 * W
wf = pr[:o1].reshape(W, 2)
blk = pr[o1:o2].reshape(B, 8)
cyc = pr[o3:o4].reshape(W, 4)
tx = pr[o4:o4 + 8 * B].reshape(B, 8)
t0 = blk[:, 3].min()
off = s.wf_fut_off.astype(np.int64)
rows = np.diff(off)
end = (wf[:, 1] - t0) / 1e3
start = (wf[:, 0] - t0) / 1e3
print(f"B={B} W={W} staged p50 {np.median(blk[:, 0] - t0) / 1e3:.2f}  p2 end max {(blk[:, 7] - t0).max() / 1e3:.2f}")
for w in np.argsort(-end)[:14]:
    c = cyc[w]
    print(f"wf {w:5d} rows {rows[w]:4d} start {start[w]:6.2f} end {end[w]:6.2f} dur {end[w] - start[w]:6.2f} "
          f"edge/round/rest cyc {c[0]:7d} {c[1]:7d} {c[2]:7d}  wait_cyc {c[3] >> 32:7d} rounds {c[3] & 0xFFFF}")
n = max(tx[:, 5].sum(), 1)
print(f"transfers {tx[:, 5].sum()}: cyc/transfer edges {tx[:, 0].sum() / n:.0f} iface {tx[:, 1].sum() / n:.0f} "
      f"settle {tx[:, 2].sum() / n:.0f} store {tx[:, 3].sum() / n:.0f}  iters/transfer {tx[:, 4].sum() / n:.1f} "
      f"K mean {tx[:, 6].sum() / n:.2f} k mean {tx[:, 7].sum() / n:.2f}")
lb = np.argsort(-(blk[:, 7] - t0))[:6]
for b in lb:
    print(f"blk {b}: staged {(blk[b, 0] - t0) / 1e3:.2f} p2end {(blk[b, 7] - t0) / 1e3:.2f} end {(blk[b, 2] - t0) / 1e3:.2f} "
          f"transfers {tx[b, 5]} cyc e/i/s/st {tx[b, 0]} {tx[b, 1]} {tx[b, 2]} {tx[b, 3]}")
# which workflows ran in the slowest block: those whose [start,end] lie in it -- by the host rule
k4 = pr[o2:o3].reshape(R, 8)
k1_end = blk[:, 2].max()
names = ["start", "n_adm", "tables", "done", "waited", "prefix", "pass1", "loads"]
print("K4 stamps, us after K1 end (median / max over resources):")
for j in (0, 4, 7, 1, 2, 5, 6, 3):
    v = k4[:, j]
    v = v[(v > 0) & (v < (1 << 62))]
    if len(v):
        d = (v - k1_end) / 1e3
        print(f"  {names[j]:7s} med {np.median(d):6.2f} max {d.max():6.2f} n {len(v)}")
bw = nalar.nalar_debug_blocks(ctx.h).astype(np.int64)
blk_of = np.searchsorted(bw, np.arange(W), side="right") - 1
maxd = None
try:
    from oracle import oracle_epoch
    maxd = oracle_epoch(s, "srtf")["wf_agg"][:, 8]
except Exception:
    pass
print("slowest blocks (p2 end), their workflows: rows/depth start-end us wait_kcyc")
for b in np.argsort(-(blk[:, 7] - t0))[:5]:
    ws = range(bw[b], bw[b + 1])
    desc = "  ".join(f"{rows[w]}/{maxd[w] if maxd is not None else '?'} {start[w]:.1f}-{end[w]:.1f} w{(cyc[w, 3] >> 32) // 1000}"
                     for w in ws)
    print(f" blk {b} p2end {(blk[b, 7] - t0) / 1e3:.2f} rows {off[bw[b + 1]] - off[bw[b]]}: {desc}")
