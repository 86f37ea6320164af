#!/usr/bin/env python
"""Benchmark of the policy epoch: futures/s and epoch latency (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--impl nalar|reference]

Workload: the SWE-recursive future table (SURVEY §8(d) C4/C5 recipe, DESIGN.md
"Input recipe") with 2^17 futures per GPU -- at N=1 exactly the paper-scale
C4 table (131,072 futures, 64 instances, state affinity), at N=8 the C5 scale-
out table (2^20 futures) sharded by workflow id.  One step = one policy epoch
(SRTF, the paper's scalability policy) over the whole table:
K1 sweep -> [NCCL allreduce] -> K4 assign.  Inputs are resident in HBM before
the timed region; L2 is flushed (256 MB memset, untimed) before every epoch.
Under torchrun each rank owns one shard, NCCL carries the per-epoch exchange.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FUT_PER_GPU = 1 << 17
METRIC = "futures scheduled/sec and policy-epoch latency at 130K futures, 1/2/4/8 B200"


def nearest_rank(xs, q):
    xs = sorted(xs)
    if not xs:
        return None
    k = max(1, int(np.ceil(q / 100.0 * len(xs))))
    return xs[k - 1]


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_table(n_gpus, seed):
    from nalar_gen import swe_table
    return swe_table(n_gpus * FUT_PER_GPU, seed=seed, name="C4" if n_gpus == 1 else "C5")


def workload_config(n_gpus, table, policy, collective="peer"):
    return {"workload": ("C4 paper-scale SWE-recursive future table" if n_gpus == 1 else
                         f"C5 scale-out SWE-recursive table sharded by workflow id over {n_gpus} GPUs"),
            "futures_total": table.n_futures, "futures_per_gpu": FUT_PER_GPU,
            "workflows": table.n_workflows, "edges": table.n_edges,
            "instances": table.n_instances, "types": table.n_types, "policy": policy.upper(),
            "levels": 256, "l2": "flushed between epochs (256 MB memset, untimed)",
            "parallelism": f"workflow-sharded x{n_gpus}" + (
                (" + peer-memory slot exchange (k_peer)" if collective == "peer" else " + NCCL allreduce")
                if n_gpus > 1 else ""),
            "recipe_deviation": "generator drift from SURVEY §8(d) C4 (DESIGN.md §6): base_load U{0..4} "
                                "(survey U{0..16}), rounds R = min(8, Geometric(0.48)) (survey 1 + "
                                "Geometric(0.3), cap 8); the benched table is the parity-tested one; "
                                "the recipe as written is timed as c4_survey_recipe (N=1)"}


def profile_spans(nalar, make_ctx, s, pol, flush, n=8):
    """Device-side durations from %globaltimer stamps (NALAR_F_PROFILE, direct
    launches, L2 flushed before each epoch, mean over n epochs): K1 = first
    block entry to last block end, K4 = its first block start to last block
    end, the last workflow's end, K4's end after K1's."""
    import torch
    pctx = make_ctx(nalar.NALAR_F_PROFILE | nalar.NALAR_F_NO_GRAPH)
    pctx.upload(s)
    st = torch.cuda.ExternalStream(pctx.stream)
    W, R = s.n_workflows, s.n_instances + s.n_types
    acc = {}
    for i in range(n + 2):
        with torch.cuda.stream(st):
            flush.zero_()
        pctx.epoch(pol)
        torch.cuda.synchronize()
        if i < 2:
            continue
        pr = nalar.nalar_debug_profile(pctx.h).astype(np.int64)
        B = (len(pr) - 2 * W - 8 * R - 4 * W) // 16
        wfp = pr[:2 * W].reshape(W, 2)
        blk = pr[2 * W:2 * W + 8 * B].reshape(B, 8)
        k4p = pr[2 * W + 8 * B:2 * W + 8 * B + 8 * R].reshape(R, 8)
        t0, k1_end = blk[:, 3].min(), blk[:, 2].max()
        k4s = k4p[:, 0][k4p[:, 0] > 0]
        vals = {"k1_span": (k1_end - t0) / 1e3,
                "k1_staging_max": (blk[:, 0] - blk[:, 3]).max() / 1e3,
                "last_workflow_end": (wfp[:, 1].max() - t0) / 1e3,
                "k1_tail_after_last_workflow": (k1_end - wfp[:, 1].max()) / 1e3,
                "k4_span": (k4p[:, 3].max() - k4s.min()) / 1e3 if len(k4s) else None,
                "k4_end_after_k1": (k4p[:, 3].max() - k1_end) / 1e3,
                "k4_pdl_release_after_k1": (k4p[:, 4].min() - k1_end) / 1e3}
        for k, v in vals.items():
            if v is not None:
                acc.setdefault(k, []).append(float(v))
    pctx.close()
    return {k: float(np.mean(v)) for k, v in acc.items()}


def oracle_time(s, policy, budget_s, min_runs=1, max_runs=10**6):
    """Time the CPU oracle as it stands on one host core: O1-O9 timed inside C
    (oracle_epoch_times: CLOCK_MONOTONIC around the epoch function only, no
    ctypes marshalling or output allocation), in chunks of 5 runs until the
    budget is spent.  Returns seconds per run."""
    from oracle import oracle_epoch_times
    try:
        cpus = sorted(os.sched_getaffinity(0))
        os.sched_setaffinity(0, {cpus[-1]})
    except Exception:
        cpus = None
    times = []
    t_end = time.perf_counter() + budget_s
    while (len(times) < min_runs or time.perf_counter() < t_end) and len(times) < max_runs:
        times.extend(oracle_epoch_times(s, policy, min(5, max_runs - len(times))).tolist())
    if cpus:
        os.sched_setaffinity(0, set(cpus))
    return times


def cpu_model():
    """lscpu model name and the host's logical CPU count."""
    name = "unknown"
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                name = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return f"{name} (lscpu), nproc {os.cpu_count()}"


class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except Exception:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def survey_bytes(s, n_elig):
    """SURVEY §8(d) byte model as written: 22 B per future (fixed inputs 12,
    written depth / flags 3, outputs 4, ...), 7 B per edge (4 B edge list + 3 B
    predecessor state / depth gathers), 40 B per workflow, 7 B per eligible
    future (rank traffic)."""
    return 22 * s.n_futures + 7 * s.n_edges + 40 * s.n_workflows + 7 * n_elig


def k1_algorithmic_bytes(s, n_elig):
    """SURVEY §8(d) byte model recomputed for this layout:
    per future 11 B read (state, type, round, executor, pin, edge_off) + 7 B
    written (status, level, depth, instance, new_pin); 4 B per edge; per
    workflow 48 B (offset, prio, 10 aggregates) + 4 B per (workflow, type) of
    K,V hints (hint, level, home); 8 B per eligible item."""
    return (18 * s.n_futures + 4 * s.n_edges + 48 * s.n_workflows + 4 * s.n_workflows * s.n_types +
            8 * n_elig)


def k4_algorithmic_bytes(R, levels, G, n_elig, n_asg):
    return 4 * R * levels * G + 8 * n_elig + 10 * n_asg


def load_traffic(kernel):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(kernel)
    except Exception:
        return None


def c3_dynamic(nalar, device, epochs, warm=450, seed=1):
    """BASELINE config 3: the router workflow at 80 RPS (nalar_gen.dynamic), one
    epoch every 100 ms of simulated time.  Per epoch through the public API:
    the epoch, the fetch of the decisions the simulator needs, and the delta
    (apply-assigned, updates, retirements, appends) applied on the device.
    The simulator's own Python step is excluded from the timed region."""
    from nalar_gen import RouterSim
    sim = RouterSim(seed)
    sim.warmup(warm)
    s = sim.snapshot()
    import torch
    ctx = nalar.Context(200000, 400000, 20000, 32, 4, device=device)
    ctx.upload(s)
    keep = []

    def pinned(n, dt):                   # reservation-sized pinned outputs: the one-kernel fetch
        t = torch.empty(max(n * np.dtype(dt).itemsize, 1), dtype=torch.uint8, pin_memory=True)
        keep.append(t)
        return t.numpy()[:n * np.dtype(dt).itemsize].view(dt)
    outb = {"new_pin": pinned(200000, np.uint8), "assign_row": pinned(200000, np.uint32),
            "assign_inst": pinned(200000, np.int16)}
    lat, live, app, upd, ret = [], [], [], [], []
    warm_epochs = 5                      # untimed: first-delta buffer allocation, graph capture
    for k in range(warm_epochs + epochs):
        t0 = time.perf_counter()
        ctx.epoch("srtf")
        r = ctx.fetch(("new_pin", "assign"), out=outb)
        r["new_pin"] = r["new_pin"][:ctx.n[0]]
        t1 = time.perf_counter()
        d = sim.step(r["assign_row"], r["assign_inst"], r["new_pin"])
        t2 = time.perf_counter()
        ctx.apply_delta(d)
        t3 = time.perf_counter()
        if k < warm_epochs:
            continue
        lat.append((t1 - t0) + (t3 - t2))
        live.append(d.n_futures_after); app.append(len(d.app_wf_id))
        upd.append(len(d.upd_seq)); ret.append(len(d.retired_wf_id))
    ctx.close()
    ms = [x * 1e3 for x in lat]
    return {"workload": "C3 router workflow, 80 RPS Poisson arrivals, 100 ms epochs, dynamic control flow",
            "epochs": epochs, "warmup_epochs": warm_epochs, "live_futures_mean": float(np.mean(live)),
            "appended_per_epoch": float(np.mean(app)), "updates_per_epoch": float(np.mean(upd)),
            "retired_workflows_per_epoch": float(np.mean(ret)),
            "epoch_fetch_delta_ms_p50": nearest_rank(ms, 50), "epoch_fetch_delta_ms_p99": nearest_rank(ms, 99),
            "futures_per_s": float(np.mean(live)) / (nearest_rank(ms, 50) / 1e3)}


def run_reference(args, world, rank):
    """--impl reference: the oracle (this tier's reference arm) on host cores."""
    if rank != 0:
        return
    table = make_table(world, args.seed)
    from oracle import build_oracle
    build_oracle()
    if args.warmup:
        oracle_time(table, args.policy, 0, min_runs=args.warmup, max_runs=args.warmup)
    times = oracle_time(table, args.policy, 0, min_runs=args.steps, max_runs=args.steps)
    mean = float(np.mean(times))
    value = table.n_futures / mean
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "futures/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": workload_config(world, table, args.policy),
            "cpu_baseline": {"value": value, "unit": "futures/s", "cores": 1, "kind": "oracle",
                             "sample": f"full table ({table.n_futures} futures) x {args.steps} epochs, "
                                       f"single-threaded C oracle (gcc -O2), O1-O9 timed inside C, on 1 "
                                       f"core of {cpu_model()}"},
            "e2e": {"value": value, "unit": "futures/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "epoch_ms_p50": nearest_rank([t * 1e3 for t in times], 50),
            "epoch_ms_p99": nearest_rank([t * 1e3 for t in times], 99)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="nalar", choices=["nalar", "reference"])
    ap.add_argument("--policy", default="srtf", choices=["fcfs", "srtf", "lpt"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--c3-epochs", type=int, default=60)
    ap.add_argument("--c5", type=int, default=1, help="also time the 2^20-future C5 table at N=1 (c5_g1)")
    ap.add_argument("--c4-survey", type=int, default=1,
                    help="also time C4 generated with SURVEY 8(d)'s recipe as written (c4_survey_recipe)")
    ap.add_argument("--collective", default="nccl", choices=["peer", "nccl"],
                    help="rank exchange for N > 1: the library's NCCL allreduce (default; the "
                         "north_star's collective), or kernels storing into peer memory (CUDA IPC)")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if world == 1:
        world = 1
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")       # one node: bootstrap over loopback
    import torch
    import torch.distributed as dist
    from paper_2601_05109_b200 import nalar
    from paper_2601_05109_b200.sharding import shard_bounds

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    table = make_table(world, args.seed)
    w0, w1 = shard_bounds(table.wf_fut_off, world)[rank]
    s = table.slice_workflows(w0, w1) if world > 1 else table
    pol = nalar.POLICIES[args.policy]

    nccl_id = None
    if world > 1:
        obj = [nalar.nalar_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    coll = args.collective

    def new_ctx(flags=0):
        nonlocal coll
        mk = lambda c: nalar.Context(max(s.n_futures, 1), max(s.n_edges, 1), max(s.n_workflows, 1),  # noqa: E731
                                     s.n_instances, s.n_types, device=local, rank=rank, world=world,
                                     nccl_id=nccl_id, flags=flags, collective=c)
        if world == 1 or coll == "nccl":
            return mk(None)
        # peer memory over CUDA IPC; every rank falls back to NCCL if any rank cannot open a peer
        from paper_2601_05109_b200.sharding import connect_peers
        c, ok = mk(nalar.NALAR_COLL_PEER), 1
        try:
            connect_peers(c)
        except nalar.NalarError as e:
            print(f"[bench] rank {rank}: peer connect failed ({e}); using NCCL", file=sys.stderr)
            ok = 0
        t = torch.tensor([ok], dtype=torch.int32, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()):
            return c
        c.close()
        coll = "nccl"
        return mk(None)

    ctx = new_ctx()
    ctx.upload(s)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        if world > 1:
            dist.barrier()

    def timed_epochs(n, do_flush, clocks=None):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(n)]
        barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for a, b in ev:
                if do_flush:
                    flush.zero_()
                a.record(stream)
                ctx.epoch(pol)
                b.record(stream)
        torch.cuda.synchronize()
        barrier()
        t = torch.tensor([a.elapsed_time(b) for a, b in ev], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.cpu().numpy()

    # warm-up (also builds the CUDA graph)
    timed_epochs(args.warmup, True)
    with ClockSampler(local) as clk:
        ms = timed_epochs(args.steps, True)
    ms_warm = timed_epochs(args.steps, False)
    st = ctx.stats()
    mean_ms = float(np.mean(ms))
    total_fut = table.n_futures
    value = total_fut / (mean_ms / 1e3)

    # NEXT rows in the same timed configuration: resource
    # reassignment (NEXT-2) switched on; K,V hints (NEXT-3) are always computed
    ctx.set_policy_params(reassign=True, u_hi_pct=80, u_lo_pct=30)
    timed_epochs(args.warmup, True)
    ms_ra = timed_epochs(max(args.steps // 4, 10), True)
    ra_out = ctx.fetch(("reassign", "kv"))
    ctx.set_policy_params(reassign=False)
    # HoL migration (NEXT-1): the same table with synthetic wait ages /
    # head-job times (nalar_gen.with_hol_inputs on the global table, then this
    # rank's shard; SPEC delta = 2)
    mig = {}
    if True:
        from nalar_gen import with_hol_inputs
        sh = with_hol_inputs(table)
        sh = sh.slice_workflows(w0, w1) if world > 1 else sh
        ctx.set_policy_params(migrate=True, theta_wait=50, theta_head=50, delta=2)
        ctx.upload(sh)
        timed_epochs(args.warmup, True)
        ms_mig = timed_epochs(max(args.steps // 4, 10), True)
        mo = ctx.fetch(("migrate",))
        ctx.set_policy_params(migrate=False)
        ctx.upload(s)
        mig = {"migrate_on_epoch_us": float(np.mean(ms_mig)) * 1e3, "migrated": int(mo["n_migrated"])}
        # batch coalescing (NEXT-4): max_batch 4 on the NONE-affinity types,
        # three methods drawn per future (global table, then this rank's shard)
        sb = table.copy()
        sb.f_method = np.random.default_rng(3).integers(0, 3, table.n_futures).astype(np.uint8)
        sb = sb.slice_workflows(w0, w1) if world > 1 else sb
        ctx.set_policy_params(t_max_batch=np.where(s.t_affinity == 0, 4, 0), n_types=s.n_types)
        ctx.upload(sb)
        timed_epochs(args.warmup, True)
        ms_b = timed_epochs(max(args.steps // 4, 10), True)
        bo = ctx.fetch(("batch",))
        ctx.set_policy_params()
        ctx.upload(s)
        mig.update({"batch_on_epoch_us": float(np.mean(ms_b)) * 1e3, "batches": int(bo["n_batches"])})
    next_rows = {"reassign_on_epoch_us": float(np.mean(ms_ra)) * 1e3,
                 "reassign_commands": int(ra_out["n_reassign"]), **mig,
                 "kv_hints": {k: int(v) for k, v in zip(("none", "retain", "offload", "drop"),
                                                       np.bincount(ra_out["kv_hint"].ravel(), minlength=4))}}

    # per-kernel device durations from %globaltimer stamps (NALAR_F_PROFILE, a
    # separate untimed context, L2 flushed, mean of 8 epochs): K1 span, K4
    # span, the last workflow's end, K4 after K1 -- single rank
    crit = profile_spans(nalar, lambda f: new_ctx(flags=f), s, pol, flush) if world == 1 else {}

    # the same per kernel from CUDA event nodes captured inside the epoch graph
    # (they perturb the graph a little: a cross-check, not the roofline input)
    tctx = new_ctx(flags=nalar.NALAR_F_TIMING)
    tctx.upload(s)
    k1, k4, coll = [], [], []
    tstream = torch.cuda.ExternalStream(tctx.stream)
    for i in range(args.warmup + args.steps):
        with torch.cuda.stream(tstream):
            flush.zero_()
        tctx.epoch(pol)
        ts = tctx.stats()
        if i >= args.warmup:
            k1.append(ts.k1_us); k4.append(ts.k4_us); coll.append(ts.coll_us)
    tctx.close()
    k1_us, k4_us, coll_us = float(np.mean(k1)), float(np.mean(k4)), float(np.mean(coll))
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"

    def roofline_of(tab, n_elig, k1_dev_us, k1_ev_us):
        """K1 (the dominant kernel) against HBM: SURVEY §8(d) bytes as written
        (primary) and DESIGN §4's layout bytes, over K1's device duration."""
        bs, bl = survey_bytes(tab, n_elig), k1_algorithmic_bytes(tab, n_elig)
        ach = bs / (k1_dev_us * 1e-6) / 1e9
        out = {"bound": "hbm", "kernel": "k1_sweep", "achieved": ach, "peak": peak, "unit": "GB/s",
               "frac": ach / peak, "traffic": None, "algorithmic_bytes": bs,
               "algorithmic_bytes_model": "SURVEY §8(d): 22 B/future + 7 B/edge + 40 B/workflow + "
                                          "7 B/eligible future",
               "layout_bytes": bl, "layout_frac": bl / (k1_dev_us * 1e-6) / 1e9 / peak,
               "duration_us": k1_dev_us,
               "duration_source": "%globaltimer span of K1 (first block entry to last block end), "
                                  "mean of 8 L2-flushed epochs",
               "peak_source": peak_src}
        if k1_ev_us:
            out["achieved_events"] = bs / (k1_ev_us * 1e-6) / 1e9
        return out
    k1_dev = crit.get("k1_span") or k1_us
    roof = roofline_of(s, st.n_eligible, k1_dev, k1_us)
    roof["traffic"] = load_traffic("k1_sweep")

    # end to end through the public API: pinned host table -> nalar_step
    # (H2D + validate, epoch, D2H of the decisions, one synchronisation),
    # every step; the split calls (upload / epoch / fetch) timed beside it
    keep = []

    def pinned_like(a):
        t = torch.empty(max(a.nbytes, 1), dtype=torch.uint8, pin_memory=True)
        keep.append(t)
        v = t.numpy()[:a.nbytes].view(a.dtype).reshape(a.shape)
        v[...] = a
        return v
    from nalar_gen import Snapshot
    sp = Snapshot(global_row_base=s.global_row_base, name=s.name,
                  **{k: pinned_like(a) for k, a in s.arrays().items()})
    h2d = sum(a.nbytes for a in sp.arrays().values())

    def pin_alloc(n, dt):
        return pinned_like(np.zeros(n, dt))
    # the decisions a controller acts on: status, instance, the ordered
    # assignment list, new_pin (SESSION homes to record, Q13) and level
    E2E_FIELDS = ("status", "level", "instance", "new_pin", "assign")
    outb = ctx.output_buffers(E2E_FIELDS, alloc=pin_alloc)
    e2e_t, split_t = [], []
    n_asg = 0
    for i in range(3 + args.e2e_steps):
        barrier()
        t0 = time.perf_counter()
        r = ctx.step(sp, pol, E2E_FIELDS, out=outb)
        dt = time.perf_counter() - t0
        n_asg = r["n_assigned"]
        streamed = ctx.last_step_streamed()
        if i >= 3:
            e2e_t.append(dt)
    for i in range(3 + args.e2e_steps):
        barrier()
        t0 = time.perf_counter()
        ctx.upload(sp)
        ctx.epoch(pol)
        ctx.fetch(E2E_FIELDS, out=outb)
        if i >= 3:
            split_t.append(time.perf_counter() - t0)
    # where the e2e step goes (separately timed, wall clock, same buffers)
    parts = {"upload": [], "epoch_sync": [], "fetch": []}
    for i in range(3 + min(args.e2e_steps, 20)):
        t0 = time.perf_counter()
        ctx.upload(sp)
        t1 = time.perf_counter()
        ctx.epoch(pol)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ctx.fetch(E2E_FIELDS, out=outb)
        t3 = time.perf_counter()
        if i >= 3:
            parts["upload"].append(t1 - t0); parts["epoch_sync"].append(t2 - t1); parts["fetch"].append(t3 - t2)
    e2e_parts = {k + "_us_p50": float(np.median(v) * 1e6) for k, v in parts.items()}
    et = torch.tensor(e2e_t, dtype=torch.float64)
    if world > 1:
        et = et.cuda()
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_mean = float(et.cpu().mean())
    d2h = 5 * s.n_futures + 6 * n_asg + 4 * 9   # status, level, new_pin (1 B), instance (2 B); list; counters

    line = {"metric": METRIC, "value": value, "unit": "futures/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": workload_config(world, table, args.policy, coll),
            "epoch_us_p50": nearest_rank(list(ms * 1e3), 50),
            "epoch_us_p99": nearest_rank(list(ms * 1e3), 99),
            "warm_l2": {"ms_per_step": float(np.mean(ms_warm)),
                        "value": total_fut / (float(np.mean(ms_warm)) / 1e3)},
            "kernels_us": {"k1_sweep": crit.get("k1_span", k1_us), "k4_assign": crit.get("k4_span", k4_us),
                           "k4_end_after_k1": crit.get("k4_end_after_k1"),
                           "exchange": (coll_us if world > 1 else None),
                           "source": ("%globaltimer spans (profile context)" if crit else "CUDA events"),
                           "events": {"k1_sweep": k1_us, "k4_assign": k4_us,
                                      "exchange": (coll_us if world > 1 else None)}},
            "counts": {"ready": st.n_ready, "eligible": st.n_eligible, "assigned": st.n_assigned,
                       "doomed": st.n_doomed},
            "roofline": roof,
            "e2e": {"value": total_fut / e2e_mean, "unit": "futures/s", "ms_per_step": e2e_mean * 1e3,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "api": "nalar_step",
                    "fields": list(E2E_FIELDS), "streamed": streamed,
                    "split_calls_ms_per_step": float(np.mean(split_t) * 1e3), "parts": e2e_parts},
            # per epoch: k_zero (exchange buffer + counters), k1_sweep, k4_assign
            "gpu_launches": 3 * args.steps,
            "next_rows": next_rows,
            "critical_path_us": crit,
            "clocks": clk.summary(),
            "paper_context": "464 ms per global-control-loop at 131K futures, Python+gRPC+Redis on "
                             "64 emulated CPU nodes (PAPER.md:715); context, not the target"}
    if rank == 0 and world == 1 and args.c3_epochs:
        line["c3_dynamic"] = c3_dynamic(nalar, local, args.c3_epochs)
    if world == 1 and args.c5:
        # BASELINE config 5 at G = 1: the 2^20-future C5 table on one B200 -- the
        # bandwidth-meaningful size; epochs timed like the C4 line
        from nalar_gen import c5
        s5 = c5(args.seed)
        c5ctx = nalar.Context.for_snapshot(s5, device=local)
        c5ctx.upload(s5)
        st5s = torch.cuda.ExternalStream(c5ctx.stream)
        n5 = min(args.steps, 300)
        ev5 = []
        with torch.cuda.stream(st5s):
            for i in range(max(args.warmup, 3) + n5):
                flush.zero_()
                a5, b5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a5.record(st5s)
                c5ctx.epoch(pol)
                b5.record(st5s)
                if i >= max(args.warmup, 3):
                    ev5.append((a5, b5))
        torch.cuda.synchronize()
        us5 = [a5.elapsed_time(b5) * 1e3 for a5, b5 in ev5]
        st5 = c5ctx.stats()
        c5ctx.close()
        sp5 = profile_spans(nalar, lambda f: nalar.Context.for_snapshot(s5, device=local, flags=f), s5, pol,
                            flush, n=4)
        line["c5_g1"] = {"workload": "C5 SWE-recursive table, 2^20 futures, one B200 (BASELINE config 5, G=1)",
                         "futures": s5.n_futures, "workflows": s5.n_workflows, "edges": s5.n_edges,
                         "epochs": n5, "epoch_us_mean": float(np.mean(us5)),
                         "epoch_us_p50": nearest_rank(us5, 50), "epoch_us_p99": nearest_rank(us5, 99),
                         "value": s5.n_futures / (float(np.mean(us5)) * 1e-6), "unit": "futures/s",
                         "counts": {"ready": st5.n_ready, "eligible": st5.n_eligible,
                                    "assigned": st5.n_assigned, "doomed": st5.n_doomed},
                         "kernels_us": sp5,
                         "roofline": roofline_of(s5, st5.n_eligible, sp5.get("k1_span"), None)}
        line["c5_g1"]["roofline"]["traffic"] = load_traffic("k1_sweep_c5")
    if rank == 0 and world == 1 and args.c4_survey:
        # C4 generated with SURVEY §8(d)'s recipe as written (base_load
        # U{0..16}, rounds 1 + Geometric(0.3)) beside the benched, parity-tested
        # generator (DESIGN.md §6 states the drift); same timing as the C4 line;
        # its parity with the oracle is tests/test_parity_gpu.py::test_c4_survey_recipe
        from nalar_gen import swe_table
        sv = swe_table(1 << 17, args.seed, recipe="survey")
        svctx = nalar.Context.for_snapshot(sv, device=local)
        svctx.upload(sv)
        svs = torch.cuda.ExternalStream(svctx.stream)
        nsv = min(args.steps, 500)
        evs = []
        with torch.cuda.stream(svs):
            for i in range(max(args.warmup, 3) + nsv):
                flush.zero_()
                a6, b6 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a6.record(svs)
                svctx.epoch(pol)
                b6.record(svs)
                if i >= max(args.warmup, 3):
                    evs.append((a6, b6))
        torch.cuda.synchronize()
        ussv = [x.elapsed_time(y) * 1e3 for x, y in evs]
        stsv = svctx.stats()
        svctx.close()
        line["c4_survey_recipe"] = {
            "workload": "C4 with SURVEY 8(d)'s generator recipe as written (base_load U{0..16}, "
                        "rounds 1 + Geometric(0.3), cap 8)",
            "futures": sv.n_futures, "workflows": sv.n_workflows, "edges": sv.n_edges, "epochs": nsv,
            "epoch_us_mean": float(np.mean(ussv)), "epoch_us_p50": nearest_rank(ussv, 50),
            "epoch_us_p99": nearest_rank(ussv, 99), "value": sv.n_futures / (float(np.mean(ussv)) * 1e-6),
            "unit": "futures/s",
            "counts": {"ready": stsv.n_ready, "eligible": stsv.n_eligible, "assigned": stsv.n_assigned,
                       "doomed": stsv.n_doomed}}
    if rank == 0 and world == 1:
        from oracle import build_oracle
        build_oracle()
        times = oracle_time(table, args.policy, args.cpu_budget, min_runs=5)
        med = float(np.median(times))
        line["cpu_baseline"] = {"value": table.n_futures / med, "unit": "futures/s",
                                "cores": 1, "kind": "oracle", "statistic": "median",
                                "epoch_ms_median": med * 1e3, "epoch_ms_mean": float(np.mean(times)) * 1e3,
                                "sample": f"C4 full table ({table.n_futures} futures) x {len(times)} "
                                          f"epochs (~{args.cpu_budget:.0f} s budget), single-threaded C "
                                          f"oracle (gcc -O2), O1-O9 timed inside C, pinned to 1 core of "
                                          f"{cpu_model()}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
