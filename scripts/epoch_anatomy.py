"""Where does the epoch go?  Epoch time (graph replay, L2 flushed, CUDA events)
and the K1 / K4 critical-path stamps (NALAR_F_PROFILE, separate context) on
several table variants: C1 (pure overhead), C2, C4 with and without the deep
workflows.

  python scripts/epoch_anatomy.py [--epochs 200] [--out gpurun_out/anatomy.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import c1, c2, swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--epochs", type=int, default=200)
ap.add_argument("--out", default="gpurun_out/anatomy.json")
ap.add_argument("--only", default="")
a = ap.parse_args()

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def epoch_us(s, n):
    ctx = nalar.Context.for_snapshot(s)
    ctx.upload(s)
    st = torch.cuda.ExternalStream(ctx.stream)
    out = []
    with torch.cuda.stream(st):
        for i in range(n + 10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ctx.epoch("srtf")
            e1.record(st)
            out.append((e0, e1))
    torch.cuda.synchronize()
    ctx.close()
    t = np.array([x.elapsed_time(y) for x, y in out[10:]]) * 1e3
    return float(t.mean()), float(np.percentile(t, 50))


def stamps(s):
    ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_PROFILE | nalar.NALAR_F_NO_GRAPH)
    ctx.upload(s)
    for _ in range(3):
        with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream)):
            flush.zero_()
        ctx.epoch("srtf")
    torch.cuda.synchronize()
    pr = nalar.nalar_debug_profile(ctx.h).astype(np.int64)
    ctx.close()
    W, R = s.n_workflows, s.n_instances + s.n_types
    B = (len(pr) - 2 * W - 8 * R - 4 * W) // 16
    wf = pr[:2 * W].reshape(W, 2)
    blk = pr[2 * W:2 * W + 8 * B].reshape(B, 8)
    k4 = pr[2 * W + 8 * B:2 * W + 8 * B + 8 * R].reshape(R, 8)
    t0 = blk[:, 3].min()
    k1_end = blk[:, 2].max()
    p2_end = blk[:, 7] - t0          # after the P2 barrier (+ griddepcontrol.wait)
    pct = lambda x: [float(np.percentile(x, q)) / 1e3 for q in (0, 50, 90, 100)]  # noqa: E731
    return {"blocks": int(B), "k1_span_us": float(k1_end - t0) / 1e3,
            "staged_us_pct": pct(blk[:, 0] - t0),
            "p2_end_us_pct": pct(p2_end),
            "p3_body_us_pct": pct(blk[:, 4] - blk[:, 7]),
            "p4_us_pct": pct(blk[:, 5] - blk[:, 4]),
            "p5_us_pct": pct(blk[:, 2] - blk[:, 5]),
            "block_end_us_pct": pct(blk[:, 2] - t0),
            "last_wf_end_us": float(wf[:, 1].max() - t0) / 1e3,
            "k4_start_after_k1_us": float(k4[:, 0].min() - k1_end) / 1e3,
            "k4_release_after_k1_us": float(k4[:, 4].min() - k1_end) / 1e3,
            "k4_end_after_k1_us": float(k4[:, 3].max() - k1_end) / 1e3}


tables = {"c1": c1, "c2": lambda: c2(1), "c4": lambda: swe_table(1 << 17, 1),
          "c4_nodeep": lambda: swe_table(1 << 17, 1, p_deep=0.0),
          "c4_half": lambda: swe_table(1 << 16, 1)}
res = {}
for name, mk in tables.items():
    if a.only and name not in a.only.split(","):
        continue
    s = mk()
    m, p50 = epoch_us(s, a.epochs)
    res[name] = {"N": s.n_futures, "W": s.n_workflows, "epoch_us_mean": m, "epoch_us_p50": p50, **stamps(s)}
    print(name, json.dumps(res[name]), flush=True)
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(res, open(a.out, "w"), indent=1)
