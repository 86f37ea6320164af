"""Experiment: K1 timeline on a table of deep (long) workflows only, at
different numbers per CTA -- how much of the compose step cost is contention?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from nalar_gen import configs as cf  # noqa: E402
from nalar_gen import TableBuilder  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402


def deep_table(n_wf, seed=1):
    rng = np.random.default_rng(seed)
    tb = TableBuilder(i_type=np.repeat(np.arange(8), 8), i_cap=np.full(64, 16), i_base_load=np.zeros(64),
                      t_affinity=cf.C4_AFFINITY, name="deep")
    for w in range(n_wf):
        types, rounds, deps, calls = cf._swe_workflow(rng, True)
        st = cf._draw_states(rng, deps, 0, p_fail=0.005, p_frontier=(0.3, 0.3), progress=float(rng.uniform(0.75, 1.0)))
        rows = [(int(st[j]), types[j], rounds[j], -1 if st[j] not in (1, 2) else types[j] * 8, -1,
                 [(p, False) for p in deps[j]] + [(p, True) for p in calls[j]]) for j in range(len(types))]
        tb.add_workflow(wid=w + 1, prio=0, rows=rows)
    return tb.build()


for n in (56, 142):
    s = deep_table(n)
    ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_PROFILE | nalar.NALAR_F_NO_GRAPH)
    ctx.upload(s)
    for _ in range(3):
        ctx.epoch("srtf")
    torch.cuda.synchronize()
    prof = nalar.nalar_debug_profile(ctx.h).astype(np.int64)
    W, R = s.n_workflows, s.n_instances + s.n_types
    B = (len(prof) - 2 * W - 8 * R - 4 * W) // 16
    wf = prof[:2 * W].reshape(W, 2)
    blk = prof[2 * W:2 * W + 8 * B].reshape(B, 8)
    cyc = prof[2 * W + 8 * B + 8 * R:2 * W + 8 * B + 8 * R + 4 * W].reshape(W, 4)
    t0 = blk[:, 3].min()
    dur = wf[:, 1] - wf[:, 0]
    steps = np.ceil(np.diff(s.wf_fut_off.astype(np.int64)) / 32)
    wait = cyc[:, 3] >> 32
    print(json.dumps({"n_wf": n, "blocks": int(B), "kernel_span_ns": int(blk[:, 2].max() - t0),
                      "compose_ns_per_step_mean": float(np.mean(dur / steps)),
                      "compose_cycles_per_step_excl_wait": float(np.mean((cyc[:, 0] + cyc[:, 1] + cyc[:, 2] - wait) / steps)),
                      "wait_cycles_mean": float(np.mean(wait))}))
    ctx.close()
