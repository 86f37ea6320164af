"""Quick A/B numbers for one build (NALAR_LIB_AB selects it): C4 / C4-no-deep /
C1 epoch (graph replay, L2 flushed before each, CUDA events; mean -- events tick in 0.512 us) and a
lone 158-row SWE workflow's P2 sweep (profile build, warm).
  NALAR_LIB_AB=libnalar_x.so python scripts/ab_quick.py [--epochs 300]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import c1, swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--epochs", type=int, default=300)
a = ap.parse_args()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def epoch_us(s, n):
    ctx = nalar.Context.for_snapshot(s)
    ctx.upload(s)
    st = torch.cuda.ExternalStream(ctx.stream)
    ev = []
    with torch.cuda.stream(st):
        for i in range(n + 10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ctx.epoch("srtf")
            e1.record(st)
            ev.append((e0, e1))
    torch.cuda.synchronize()
    ctx.close()
    t = np.array([x.elapsed_time(y) for x, y in ev[10:]]) * 1e3
    return round(float(np.mean(t)), 2)


def solo():
    s = swe_table(190, 3, p_deep=0.0)
    ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_PROFILE | nalar.NALAR_F_NO_GRAPH)
    ctx.upload(s)
    for _ in range(4):
        ctx.epoch("srtf")
    torch.cuda.synchronize()
    pr = nalar.nalar_debug_profile(ctx.h).astype(np.int64)
    ctx.close()
    W, R = s.n_workflows, s.n_instances + s.n_types
    B = (len(pr) - 2 * W - 8 * R - 4 * W) // 16
    wf = pr[:2 * W].reshape(W, 2)
    blk = pr[2 * W:2 * W + 8 * B].reshape(B, 8)
    t0 = blk[:, 3].min()
    w = int(np.argmax(np.diff(s.wf_fut_off)))
    return {"wf_us": round((wf[w, 1] - wf[w, 0]) / 1e3, 2), "p2end": round((blk[0, 7] - t0) / 1e3, 2),
            "end": round((blk[0, 2] - t0) / 1e3, 2)}


r = {"c4": epoch_us(swe_table(1 << 17, 1), a.epochs), "c4nd": epoch_us(swe_table(1 << 17, 1, p_deep=0.0), a.epochs),
     "c1": epoch_us(c1(), a.epochs // 2), "solo": solo()}
print(json.dumps(r))
