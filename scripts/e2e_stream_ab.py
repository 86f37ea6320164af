"""nalar_step at C4 through pinned host arrays: streamed (K1 stages from host
memory) vs the plain path (NALAR_STREAM_STEP=0 in a subprocess), wall clock.

  python scripts/e2e_stream_ab.py [--steps 200]
"""
import argparse
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--child", action="store_true")
ap.add_argument("--n", type=int, default=1 << 17)
a = ap.parse_args()
if not a.child:
    for env in ("1", "0", "1", "0"):
        r = subprocess.run([sys.executable, __file__, "--child", "--steps", str(a.steps), "--n", str(a.n)],
                           env={**os.environ, "NALAR_STREAM_STEP": env}, capture_output=True, text=True)
        print(env, r.stdout.strip(), r.stderr.strip()[-300:])
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import Snapshot, swe_table  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

s = swe_table(a.n, seed=1)
keep = []


def pinned_like(x):
    t = torch.empty(max(x.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    keep.append(t)
    v = t.numpy()[:x.nbytes].view(x.dtype).reshape(x.shape)
    v[...] = x
    return v


sp = Snapshot(global_row_base=0, name=s.name, **{k: pinned_like(v) for k, v in s.arrays().items()})
ctx = nalar.Context.for_snapshot(s)
out = ctx.output_buffers(("status", "instance", "assign"), alloc=lambda n, dt: pinned_like(np.zeros(n, dt)), like=s)
ts = []
for i in range(20 + a.steps):
    t0 = time.perf_counter()
    ctx.step(sp, "srtf", ("status", "instance", "assign"), out=out)
    if i >= 20:
        ts.append(time.perf_counter() - t0)
ts = np.array(ts) * 1e6
print(json.dumps({"streamed": ctx.last_step_streamed(), "mean_us": float(ts.mean()), "p50_us": float(np.median(ts)),
                  "min_us": float(ts.min())}))
