"""When do K1 blocks pass griddepcontrol.wait, relative to entry and to their sweep's end?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from nalar_gen import swe_table
from paper_2601_05109_b200 import nalar
s = swe_table(1 << 17, seed=1)
for flags, name in ((nalar.NALAR_F_PROFILE | nalar.NALAR_F_NO_GRAPH, "nograph"), (nalar.NALAR_F_PROFILE, "graph")):
    ctx = nalar.Context.for_snapshot(s, flags=flags)
    ctx.upload(s)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for i in range(6):
        torch.cuda.synchronize()
        flush.zero_()
        torch.cuda.synchronize()
        ctx.epoch("srtf")
    torch.cuda.synchronize()
    prof = nalar.nalar_debug_profile(ctx.h).astype(np.int64)
    W = s.n_workflows; R = s.n_instances + s.n_types
    B = (len(prof) - 2 * W - 8 * R - 4 * W) // 16
    blk = prof[2 * W:2 * W + 8 * B].reshape(B, 8)
    t0 = blk[:, 3].min()
    q = lambda x: [int(np.percentile(x, p)) for p in (0, 50, 90, 100)]
    print(name, "entry", q(blk[:, 3] - t0), "swept", q(blk[:, 1] - t0), "gdc_pass", q(blk[:, 7] - t0),
          "wait", q(blk[:, 7] - blk[:, 1]), "end", q(blk[:, 2] - t0),
          "p3", q(blk[:, 4] - blk[:, 7]), "p4", q(blk[:, 5] - blk[:, 4]), "p5", q(blk[:, 2] - blk[:, 5]))
    ctx.close()
