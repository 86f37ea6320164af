"""Workloads for compute-sanitizer (racecheck / synccheck / memcheck): every
kernel of the library on small tables, direct launches (no graph).

  compute-sanitizer --tool racecheck python scripts/sanitize.py [--cases c1,c2,mig,batch,ra,delta,io,unstaged,peer]

K0 (upload), K1 + K4 (epoch), K5 (HoL migration), K6 (batch coalescing),
K4's reassignment tail, the delta kernels KD1-KD4, the fetch / copy kernels,
K1's unstaged (HBM) path and the peer exchange (two ranks on one GPU).  Each
case also checks the decisions against the oracle, so a run under the
sanitizer is a parity run as well.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from nalar_gen import AFF_NONE, c1, c2, hol_table, random_table  # noqa: E402
from oracle import oracle_epoch  # noqa: E402
from paper_2601_05109_b200 import nalar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="c1,c2,mig,batch,ra,delta,io,unstaged,peer")
a = ap.parse_args()
F = nalar.NALAR_F_NO_GRAPH
KEYS = ("status", "level", "depth", "instance", "new_pin", "wf_agg", "assign_row", "assign_inst")


def same(o, g, tag):
    for k in KEYS:
        assert np.array_equal(np.asarray(o[k]), np.asarray(g[k])), (tag, k)


def epoch_case(s, tag, flags=F, policy="srtf"):
    ctx = nalar.Context.for_snapshot(s, flags=flags)
    ctx.upload(s)
    ctx.epoch(policy)
    same(oracle_epoch(s, policy), ctx.fetch(), tag)
    ctx.close()


cases = a.cases.split(",")
if "c1" in cases:
    for pol in ("fcfs", "srtf", "lpt"):
        epoch_case(c1(), f"c1 {pol}", policy=pol)
if "c2" in cases:
    epoch_case(c2(1, n_workflows=300), "c2")
if "unstaged" in cases:
    epoch_case(c2(2, n_workflows=200), "c2 unstaged", flags=F | nalar.NALAR_F_FORCE_UNSTAGED)
if "mig" in cases:
    s = hol_table(3, n_workflows=40, n_types=3, inst_per_type=4)
    prm = {"theta_wait": 3, "theta_head": 3, "delta": 1}
    ctx = nalar.Context.for_snapshot(s, flags=F)
    ctx.set_policy_params(migrate=True, **prm)
    ctx.upload(s)
    ctx.epoch("srtf")
    g = ctx.fetch()
    o = oracle_epoch(s, "srtf", migrate={"f_age": s.f_age, "i_head_rem": s.i_head_rem, **prm})
    assert np.array_equal(g["migrate_to"], o["migrate_to"]), "mig"
    ctx.close()
if "batch" in cases:
    s = random_table(5, n_workflows=40, max_rows=20, n_types=3, inst_per_type=(1, 3), max_cap=8, p_pin=0.2)
    s.t_affinity[:] = AFF_NONE
    s.f_method = np.random.default_rng(5).integers(0, 3, s.n_futures).astype(np.uint8)
    mb = np.array([3, 2, 4])
    ctx = nalar.Context.for_snapshot(s, flags=F)
    ctx.set_policy_params(t_max_batch=mb, n_types=s.n_types)
    ctx.upload(s)
    ctx.epoch("srtf")
    g = ctx.fetch()
    o = oracle_epoch(s, "srtf", batch={"t_max_batch": mb, "f_method": s.f_method})
    assert np.array_equal(g["batch_head"], o["batch_head"]), "batch"
    ctx.close()
if "ra" in cases:
    s = c2(3, n_workflows=300)
    ctx = nalar.Context.for_snapshot(s, flags=F)
    ctx.set_policy_params(reassign=True, u_hi_pct=60, u_lo_pct=40)
    ctx.upload(s)
    ctx.epoch("srtf")
    g = ctx.fetch()
    o = oracle_epoch(s, "srtf", reassign={"u_hi_pct": 60, "u_lo_pct": 40})
    assert np.array_equal(g["ra_kill"], o["ra_kill"]) and np.array_equal(g["ra_prov"], o["ra_prov"]), "ra"
    ctx.close()
if "delta" in cases:
    from nalar_gen import RouterSim
    sim = RouterSim(1)
    sim.warmup(60)
    s = sim.snapshot()
    ctx = nalar.Context(60000, 120000, 6000, 32, 4, flags=F)
    ctx.upload(s)
    for k in range(3):
        o = oracle_epoch(s, "srtf")
        ctx.epoch("srtf")
        same(o, ctx.fetch(), f"delta {k}")
        ctx.apply_delta(sim.step(o["assign_row"], o["assign_inst"], o["new_pin"]))
        s = sim.snapshot()
    ctx.close()
if "io" in cases:
    import torch
    s = c2(4, n_workflows=200)
    keep = []

    def pinned_like(x):
        t = torch.empty(max(x.nbytes, 1), dtype=torch.uint8, pin_memory=True)
        keep.append(t)
        v = t.numpy()[:x.nbytes].view(x.dtype).reshape(x.shape)
        v[...] = x
        return v
    from nalar_gen import Snapshot
    sp = Snapshot(global_row_base=0, name=s.name, **{k: pinned_like(x) for k, x in s.arrays().items()})
    ctx = nalar.Context.for_snapshot(s, flags=F)
    out = ctx.output_buffers(like=s, alloc=lambda n, dt: pinned_like(np.zeros(n, dt)))
    g = ctx.step(sp, "srtf", out=out)
    same(oracle_epoch(s, "srtf"), g, "io step")
    ctx.close()
if "peer" in cases:
    # the peer-memory exchange (k_peer_push / wait / gather), two ranks driven
    # by this process on one GPU, each on its own stream
    import torch
    from paper_2601_05109_b200.sharding import connect_local, shard_bounds
    s = c2(5, n_workflows=200)
    streams = [torch.cuda.Stream() for _ in range(2)]
    ctxs, shards = [], []
    for k, (w0, w1) in enumerate(shard_bounds(s.wf_fut_off, 2)):
        ctxs.append(nalar.Context.for_snapshot(s, world=2, rank=k, collective=nalar.NALAR_COLL_PEER,
                                               stream=streams[k].cuda_stream, flags=F))
        shards.append(s.slice_workflows(w0, w1))
    connect_local(ctxs)
    for c, sh in zip(ctxs, shards):
        c.upload(sh)
    for c in ctxs:
        c.epoch("srtf")
    outs = [c.fetch() for c in ctxs]
    o = oracle_epoch(s, "srtf")
    for k in ("status", "level", "instance"):
        assert np.array_equal(np.concatenate([g[k] for g in outs]), o[k]), ("peer", k)
    for c in ctxs:
        c.close()
print("sanitize workloads OK:", ",".join(cases))
