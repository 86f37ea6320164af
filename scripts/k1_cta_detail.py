"""Per-CTA K1 detail from NALAR_F_PROFILE stamps: which workflows share the
slowest CTAs, when each one starts and ends (ns from kernel entry).

  python scripts/k1_cta_detail.py [--n 131072] [--seed 1] [--top 6]
The CTA partition is recomputed here with the host rule of nalar_ctx.cu
partition() (greedy whole workflows, rows >= N/148 per CTA).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import swe_table  # noqa: E402
from oracle import oracle_epoch  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 17)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--top", type=int, default=6)
ap.add_argument("--out", default="gpurun_out/k1_cta_detail.json")
a = ap.parse_args()
s = swe_table(a.n, seed=a.seed)
ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_PROFILE | nalar.NALAR_F_NO_GRAPH)
ctx.upload(s)
for _ in range(5):
    ctx.epoch("srtf")
torch.cuda.synchronize()
prof = nalar.nalar_debug_profile(ctx.h).astype(np.int64)
W = s.n_workflows
R = s.n_instances + s.n_types
B_ = (len(prof) - 2 * W - 8 * R - 4 * W) // 16     # layout: [W][2] [B][8] [R][8] [W][4] [B][8]
o1, o2 = 2 * W, 2 * W + 8 * B_
o3, o4 = o2 + 8 * R, o2 + 8 * R + 4 * W
wf = prof[:o1].reshape(W, 2)
blk = prof[o1:o2].reshape(B_, 8)        # staged, swept, bucketed, entered, P3 done, P4 done
k4 = prof[o2:o3].reshape(R, 8)          # start, n_adm, tables, done, waited, prefix, pass1
cyc = prof[o3:o4].reshape(W, 4)         # edge loop, rounds, rest (SM cycles), round counts
tx = prof[o4:o4 + 8 * B_].reshape(B_, 8)  # transfer phases: edge, iface, settle, end, iters, n, K, k
t0 = blk[:, 3].min()
off = s.wf_fut_off.astype(np.int64)
sizes = np.diff(off)
target = max(64, (s.n_futures + 147) // 148)
cta = np.zeros(W, np.int64)
b, rows = 0, 0
for w in range(W):
    cta[w] = b
    rows += sizes[w]
    if rows >= target:
        b, rows = b + 1, 0
o = oracle_epoch(s, "srtf")
maxd = o["wf_agg"][:, 8]
end_blk = blk[:, 2] - t0
order = np.argsort(-end_blk)[:a.top]
res = {"n_cta": int(blk.shape[0]), "n_cta_host_rule": int(cta.max() + 1), "ctas": []}
for c in order:
    ws = np.nonzero(cta == c)[0]
    res["ctas"].append({
        "cta": int(c), "end_ns": int(end_blk[c]), "swept_ns": int(blk[c, 1] - t0),
        "p2_done_ns": int(blk[c, 7] - t0), "p3_done_ns": int(blk[c, 4] - t0), "p4_done_ns": int(blk[c, 5] - t0),
        "staged_ns": int(blk[c, 0] - t0),
        "transfer": {"n": int(tx[c, 5]), "cyc_edges_iface_settle_store": [int(x) for x in tx[c, :4]],
                     "iters": int(tx[c, 4]), "K_sum": int(tx[c, 6]), "k_sum": int(tx[c, 7])},
        "wfs": [{"w": int(w), "rows": int(sizes[w]), "depth": int(maxd[w]), "long": bool(sizes[w] >= 192),
                 "start": int(wf[w, 0] - t0), "end": int(wf[w, 1] - t0),
                 "cyc_edge_round_rest": [int(x) for x in cyc[w, :3]], "rounds": int(cyc[w, 3] & 0xFFFF), "wait_cyc": int(cyc[w, 3] >> 32)}
                for w in ws]})
print(json.dumps(res, indent=1))
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(res, open(a.out, "w"), indent=1)
