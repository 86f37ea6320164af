import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from nalar_gen import c4
from paper_2601_05109_b200 import nalar
s = c4()
for on in (False, True, False, True):
    ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_TIMING)
    if on:
        ctx.set_policy_params(reassign=True, u_hi_pct=80, u_lo_pct=30)
    ctx.upload(s)
    k1, k4, ep = [], [], []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.ExternalStream(ctx.stream)
    for i in range(60):
        with torch.cuda.stream(st):
            flush.zero_()
        ctx.epoch("srtf")
        x = ctx.stats()
        if i >= 10:
            k1.append(x.k1_us); k4.append(x.k4_us); ep.append(x.epoch_us)
    print("reassign" if on else "plain   ", "epoch %.1f k1 %.1f k4 %.1f" % (np.mean(ep), np.mean(k1), np.mean(k4)))
    ctx.close()
