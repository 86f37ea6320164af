"""K1 timeline from NALAR_F_PROFILE stamps: where does the sweep's critical path go?

  python scripts/k1_timeline.py [--n 131072] [--seed 1]
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
ap.add_argument("--out", default="gpurun_out/k1_timeline.json")
ap.add_argument("--reassign", action="store_true")
a = ap.parse_args()
s = swe_table(a.n, seed=a.seed)
ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_PROFILE | nalar.NALAR_F_NO_GRAPH)
if a.reassign:
    ctx.set_policy_params(reassign=True, u_hi_pct=80, u_lo_pct=30)
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
o = oracle_epoch(s, "srtf")
sizes = np.diff(s.wf_fut_off.astype(np.int64))
maxd = o["wf_agg"][:, 8]
dur = wf[:, 1] - wf[:, 0]
start = wf[:, 0] - t0
end = wf[:, 1] - t0
res = {
    "kernel_span_ns": int(blk[:, 2].max() - t0),
    "block_entry_spread_ns": int(blk[:, 3].max() - t0),
    "stage_ns_mean": float(np.mean(blk[:, 0] - blk[:, 3])), "stage_ns_max": int(np.max(blk[:, 0] - blk[:, 3])),
    "sweep_ns_max": int(np.max(blk[:, 1] - blk[:, 6])), "sweep_ns_mean": float(np.mean(blk[:, 1] - blk[:, 6])),
    "bucket_ns_max": int(np.max(blk[:, 2] - blk[:, 1])), "bucket_ns_mean": float(np.mean(blk[:, 2] - blk[:, 1])),
    "p1_ns_max": int(np.max(blk[:, 6] - blk[:, 0])), "stage_to_p1_ns_max": int(np.max(blk[:, 0] - blk[:, 3])),
    "p3_ns_max": int(np.max(blk[:, 4] - blk[:, 1])), "p3_ns_mean": float(np.mean(blk[:, 4] - blk[:, 1])),
    "gdc_wait_ns_max": int(np.max(blk[:, 7] - blk[:, 1])), "gdc_wait_ns_mean": float(np.mean(blk[:, 7] - blk[:, 1])),
    "p3_body_ns_max": int(np.max(blk[:, 4] - blk[:, 7])), "p3_body_ns_mean": float(np.mean(blk[:, 4] - blk[:, 7])),
    "p4_ns_max": int(np.max(blk[:, 5] - blk[:, 4])), "p5_ns_max": int(np.max(blk[:, 2] - blk[:, 5])),
    "p5_ns_mean": float(np.mean(blk[:, 2] - blk[:, 5])),
    "wf_dur_ns_max": int(dur.max()), "wf_dur_ns_mean": float(dur.mean()),
    "wf_end_ns_max": int(end.max()),
    "ns_per_row_mean": float(np.sum(dur) / np.sum(sizes)),
}
res["k4"] = {"start_after_k1_ns": int(k4[:, 0].min() - blk[:, 2].max()),
             "span_ns": int(k4[:, 3].max() - k4[:, 0].min()),
             "prologue_ns_max": int((k4[:, 1] - k4[:, 0]).max()),
             "tables_ns_max": int((k4[:, 2] - k4[:, 1]).max()),
             "walk_ns_max": int((k4[:, 3] - k4[:, 2]).max()),
             "start_spread_ns": int(k4[:, 0].max() - k4[:, 0].min()),
             "slowest_walk_r": int(np.argmax(k4[:, 3] - k4[:, 2])),
             "k1_end_to_k4_end_ns": int(k4[:, 3].max() - blk[:, 2].max()),
             "after_wait_to_nadm_ns_max": int((k4[:, 1] - k4[:, 4]).max()),
             "prefix_ns_max": int(np.max(np.where(k4[:, 5] > 0, k4[:, 5] - k4[:, 2], 0))),
             "pass1_ns_max": int(np.max(np.where(k4[:, 6] > 0, k4[:, 6] - k4[:, 5], 0))),
             "rest_of_walk_ns_max": int(np.max(np.where(k4[:, 6] > 0, k4[:, 3] - k4[:, 6], 0))),
             "wait_release_spread_ns": int(k4[:, 4].max() - k4[:, 4].min())}
top = np.argsort(-dur)[:10]
res["slowest"] = [{"w": int(w), "rows": int(sizes[w]), "max_depth": int(maxd[w]), "dur_ns": int(dur[w]),
                   "start_ns": int(start[w]), "cyc_edge_round_rest": [int(x) for x in cyc[w, :3]],
                   "rounds": int(cyc[w, 3] & 0xFFFF),
                   "steps_by_K": [int((cyc[w, 3] >> sh) & 0xFFF) for sh in (16, 28, 40, 52)]}
                  for w in top]
chunks = np.ceil(sizes / 32.0)
res["cycles_per_chunk"] = {"edge": float(cyc[:, 0].sum() / chunks.sum()),
                           "round": float(cyc[:, 1].sum() / chunks.sum()),
                           "rest": float(cyc[:, 2].sum() / chunks.sum())}
# regression of duration on rows and depth
A = np.stack([sizes, maxd, np.ones_like(sizes)], 1).astype(np.float64)
coef, *_ = np.linalg.lstsq(A, dur.astype(np.float64), rcond=None)
res["fit_ns"] = {"per_row": coef[0], "per_depth": coef[1], "const": coef[2]}
nt = max(int(tx[:, 5].sum()), 1)
res["transfer_steps"] = {"n": int(tx[:, 5].sum()),
                         "cycles_per_step": {k: float(tx[:, j].sum() / nt) for j, k in
                                             enumerate(("edges", "iface", "settle", "store"))},
                         "settle_iters_mean": float(tx[:, 4].sum() / nt), "K_mean": float(tx[:, 6].sum() / nt),
                         "k_mean": float(tx[:, 7].sum() / nt)}
k1_end = blk[:, 2].max()
last = np.nonzero(k4[:, 7] < 0)[0]
if len(last):
    res["k4"]["ra_last_block"] = int(last[0])
    res["k4"]["ra_pairing_end_ns"] = int((k4[last[0], 7] & ((1 << 62) - 1)) - k1_end)
    tick = np.where(k4[:, 7] > 0, k4[:, 7], 0)
    res["k4"]["ra_ticket_last_ns"] = int(tick.max() - k1_end) if tick.max() > 0 else None
res["k4"]["wait_release_after_k1_end_ns"] = int(k4[:, 4].min() - k1_end)
slow = np.argsort(-(k4[:, 3] - k1_end))[:6]
res["k4"]["slowest_ctas"] = [{"r": int(r), **{n: (int(k4[r, j] - k1_end) if k4[r, j] > 0 else None) for n, j in
                                             (("start", 0), ("released", 4), ("loaded", 7), ("n_adm", 1), ("tables", 2),
                                              ("prefix", 5), ("pass1", 6), ("done", 3))}} for r in slow]
# per block: [entered, staged, P2 end, P3 end, P4 end, P5 end] (ns from the first entry)
res["p2_end_ns_pct"] = {q: int(np.percentile(blk[:, 1] - t0, q)) for q in (0, 25, 50, 75, 90, 100)}
res["blocks"] = [[int(x) for x in (blk[b, 3] - t0, blk[b, 0] - t0, blk[b, 1] - t0, blk[b, 4] - t0, blk[b, 5] - t0,
                                   blk[b, 2] - t0)] for b in range(B_)]
print(json.dumps({k: v for k, v in res.items() if k != "blocks"}, indent=1))
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(res, open(a.out, "w"), indent=1)
