"""One SWE workflow alone on the GPU (K1 with a single block): its P2 sweep
time vs the same workflow inside the full C4 epoch -- per-step latency alone
vs in situ.   python scripts/solo_wf.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in (64, 128, 190, 400, 700):
    for seed in (3, 5):
        s = swe_table(n, seed, p_deep=0.0 if n < 300 else 1.0)
        ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_PROFILE | nalar.NALAR_F_NO_GRAPH)
        ctx.upload(s)
        res = []
        for fl in (1, 0):
            for _ in range(4):
                if fl:
                    with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream)):
                        flush.zero_()
                ctx.epoch("srtf")
            torch.cuda.synchronize()
            pr = nalar.nalar_debug_profile(ctx.h).astype(np.int64)
            W, R = s.n_workflows, s.n_instances + s.n_types
            B = (len(pr) - 2 * W - 8 * R - 4 * W) // 16
            wf = pr[:2 * W].reshape(W, 2)
            blk = pr[2 * W:2 * W + 8 * B].reshape(B, 8)
            cyc = pr[2 * W + 8 * B + 8 * R:2 * W + 8 * B + 8 * R + 4 * W].reshape(W, 4)
            t0 = blk[:, 3].min()
            w = int(np.argmax(np.diff(s.wf_fut_off)))
            res.append(f"{'cold' if fl else 'warm'}: staged {(blk[0, 0] - t0) / 1e3:.2f} wf dur {(wf[w, 1] - wf[w, 0]) / 1e3:.2f} "
                       f"p2end {(blk[0, 7] - t0) / 1e3:.2f} end {(blk[0, 2] - t0) / 1e3:.2f} cyc e/r/rest {cyc[w, 0]} {cyc[w, 1]} {cyc[w, 2]} rounds {cyc[w, 3] & 0xFFFF} wait {cyc[w, 3] >> 32}")
        ctx.close()
        rows = int(np.diff(s.wf_fut_off).max())
        print(f"n={n} seed={seed} W={s.n_workflows} rows={rows} steps={(rows + 31) // 32} | " + " | ".join(res), flush=True)
