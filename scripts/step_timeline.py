"""Device timeline of one nalar_step at C4 through pinned host arrays
(NALAR_F_PROFILE stamps, %globaltimer ns from the first K1 block entry):
staging, sweep end, K1 end, K4 end -- streamed vs plain (NALAR_STREAM_STEP=0).

  python scripts/step_timeline.py
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if "--child" not in sys.argv:
    for env in ("1", "0"):
        r = subprocess.run([sys.executable, __file__, "--child"], env={**os.environ, "NALAR_STREAM_STEP": env},
                           capture_output=True, text=True)
        print("NALAR_STREAM_STEP=" + env, r.stdout.strip(), r.stderr.strip()[-400:])
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import Snapshot, swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

s = swe_table(1 << 17, seed=1)
keep = []


def pinned_like(x):
    t = torch.empty(max(x.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    keep.append(t)
    v = t.numpy()[:x.nbytes].view(x.dtype).reshape(x.shape)
    v[...] = x
    return v


sp = Snapshot(global_row_base=0, name=s.name, **{k: pinned_like(v) for k, v in s.arrays().items()})
ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_PROFILE)
out = ctx.output_buffers(("status", "instance", "assign"), alloc=lambda n, dt: pinned_like(np.zeros(n, dt)), like=s)
res = []
for i in range(8):
    ctx.step(sp, "srtf", ("status", "instance", "assign"), out=out)
    prof = nalar.nalar_debug_profile(ctx.h).astype(np.int64)
    W = s.n_workflows
    R = s.n_instances + s.n_types
    B = (len(prof) - 2 * W - 8 * R - 4 * W) // 16
    blk = prof[2 * W:2 * W + 8 * B].reshape(B, 8)
    k4 = prof[2 * W + 8 * B:2 * W + 8 * B + 8 * R].reshape(R, 8)
    t0 = blk[:, 3].min()
    res.append({"staged_max": int(blk[:, 0].max() - t0), "staged_mean": int(blk[:, 0].mean() - t0),
                "k1_end": int(blk[:, 2].max() - t0), "k4_end": int(k4[:, 3].max() - t0)})
print(json.dumps({"streamed": ctx.last_step_streamed(), "last": res[-1],
                  "median": {k: int(np.median([r[k] for r in res[2:]])) for k in res[0]}}))
