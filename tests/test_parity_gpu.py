"""Parity of the CUDA path (through the C ABI) against the CPU oracle.

All integer: the bar is bit-exactness on every output (status, level, depth,
instance, new_pin, per-workflow aggregates, per-instance load / spare /
assigned, the ordered assignment list), at the oracle's small sizes AND at the
full BASELINE sizes (C4 = 2^17, C5 = 2^20 futures) in the configuration
bench.py times.
"""
import numpy as np
import pytest

from nalar_gen import (AFF_NONE, AFF_STATEFUL, PENDING, RESOLVED, RUNNING, Snapshot,
                       TableBuilder, c1, c2, c4, c5, random_table, swe_table)
from oracle import oracle_epoch, oracle_validate

pytestmark = pytest.mark.gpu

KEYS = ("status", "level", "depth", "instance", "new_pin", "wf_agg", "i_load", "i_spare",
        "i_assigned", "assign_row", "assign_inst", "kv_hint", "kv_level", "kv_home")


def _nalar():
    from paper_2601_05109_b200 import nalar
    return nalar


def run_gpu(s, policy="srtf", flags=0, levels=256, epochs=1):
    nalar = _nalar()
    ctx = nalar.Context.for_snapshot(s, flags=flags, levels=levels)
    ctx.upload(s)
    for _ in range(epochs):
        ctx.epoch(policy)
    out = ctx.fetch()
    out["stats"] = ctx.stats()
    ctx.close()
    return out


def assert_same(s, o, g, tag=""):
    for k in KEYS:
        a, b = np.asarray(o[k]), np.asarray(g[k])
        if a.shape != b.shape or not np.array_equal(a, b):
            bad = np.nonzero(a.reshape(-1) != b.reshape(-1))[0][:10] if a.shape == b.shape else "shape"
            raise AssertionError(f"{tag} {s.name}: '{k}' differs at {bad}: oracle "
                                 f"{a.reshape(-1)[:20] if a.size else a} gpu "
                                 f"{b.reshape(-1)[:20] if b.size else b}")


def check(s, policy="srtf", **kw):
    o = oracle_epoch(s, policy, levels=kw.get("levels", 256))
    g = run_gpu(s, policy, **kw)
    assert_same(s, o, g, f"[{policy} {kw}]")
    st = g["stats"]
    assert (st.n_ready, st.n_eligible, st.n_doomed, st.n_assigned) == \
        (o["n_ready"], o["n_eligible"], o["n_doomed"], len(o["assign_row"]))
    return o, g


@pytest.mark.parametrize("policy", ["fcfs", "srtf", "lpt"])
def test_c1(policy):
    check(c1(), policy)


@pytest.mark.parametrize("seed", range(240))
def test_random_tiny(seed):
    consistent = seed % 2 == 0
    s = random_table(seed, n_workflows=1 + seed % 7, max_rows=3 + seed % 40, n_types=1 + seed % 4,
                     inst_per_type=(0, 1 + seed % 5), max_preds=1 + seed % 4, consistent=consistent,
                     max_cap=1 + seed % 6, prio_range=(-4, 300 if seed % 5 == 0 else 8),
                     max_round=seed % 9)
    check(s, ["fcfs", "srtf", "lpt"][seed % 3], levels=[256, 16, 1, 200][seed % 4])


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("policy", ["srtf", "lpt"])
def test_c2(seed, policy):
    check(c2(seed), policy)


@pytest.mark.parametrize("seed", [1, 2])
def test_c4_full_size(seed):
    s = c4(seed)
    for pol in ("srtf", "lpt", "fcfs"):
        check(s, pol)


def test_c5_full_size():
    check(c5(1), "srtf")


@pytest.mark.parametrize("seed", [2, 3, 5, 8])
def test_many_long_workflows_per_block(seed):
    """Blocks holding several long (composed) workflows of unequal lengths:
    the transfer tickets alternate between the two early composers' steps,
    then follow the other long workflows largest first; also the adaptive
    compose threshold (the survey recipe's transfer load)."""
    for n in (24000, 50000):
        check(swe_table(n, seed, recipe="survey"), ("srtf", "lpt", "fcfs")[seed % 3])


@pytest.mark.parametrize("pol", ["srtf", "lpt", "fcfs"])
def test_c4_survey_recipe(pol):
    """C4 generated with SURVEY 8(d)'s recipe as written (base_load U{0..16},
    rounds 1 + Geometric(0.3)): bench.py's c4_survey_recipe table."""
    check(swe_table(1 << 17, 1, recipe="survey"), pol)


@pytest.mark.parametrize("flags", [2, 4, 6, 1])        # NO_GRAPH, FORCE_UNSTAGED, both, TIMING
def test_launch_variants(flags):
    check(c2(1), "srtf", flags=flags)
    check(swe_table(20000, seed=7), "lpt", flags=flags)


def test_repeated_epochs_and_reupload():
    nalar = _nalar()
    a, b = c2(1), swe_table(30000, seed=5)
    ctx = nalar.Context(40000, 60000, 4000, 64, 8)
    for s in (a, b, a):
        ctx.upload(s)
        for pol in ("srtf", "lpt", "srtf"):
            ctx.epoch(pol)
            ctx.epoch(pol)                       # idempotent: same table, same decisions
            g = ctx.fetch()
            assert_same(s, oracle_epoch(s, pol), g, "reupload")
    ctx.close()


def _single_workflow(n, seed):
    """One giant workflow (more rows than a K1 block can stage): the unstaged path."""
    rng = np.random.default_rng(seed)
    tb = TableBuilder(i_type=[0, 0, 1], i_cap=[50, 70, 30], i_base_load=[0, 3, 1],
                      t_affinity=[AFF_NONE, AFF_STATEFUL])
    rows = []
    for j in range(n):
        k = int(rng.integers(0, 3)) if j else 0
        preds = [(int(p), bool(rng.random() < 0.2)) for p in rng.integers(max(0, j - 40), j, k)] if j else []
        st = RESOLVED if j < n // 2 and rng.random() < 0.8 else PENDING
        rows.append((st, int(rng.integers(0, 2)), 0, -1, -1, preds))
    tb.add_workflow(7, 0, rows)
    return tb.build()


def test_giant_workflow_unstaged():
    check(_single_workflow(60000, 1), "srtf")


def test_edge_cases():
    # empty table
    e = TableBuilder(i_type=[0], i_cap=[3], i_base_load=[1], t_affinity=[AFF_NONE]).build()
    check(e)
    # empty workflows between non-empty ones; no instances for a type
    tb = TableBuilder(i_type=[1], i_cap=[2], i_base_load=[0], t_affinity=[AFF_NONE, AFF_NONE])
    tb.add_workflow(1, 0, [])
    tb.add_workflow(2, 0, [(PENDING, 0, 0, -1, -1, []), (PENDING, 1, 0, -1, -1, [])])
    tb.add_workflow(3, 0, [])
    check(tb.build())
    # extreme priorities and capacities; saturating depth and level
    tb = TableBuilder(i_type=[0, 0], i_cap=[0xFFFFFFFF, 5], i_base_load=[0xFFFFFFFF, 0xFFFFFFF0],
                      t_affinity=[AFF_NONE])
    tb.add_workflow(1, 2**31 - 1, [(PENDING, 0, 0, -1, -1, [])] * 3)
    tb.add_workflow(2, -2**31, [(RUNNING, 0, 0, 1, -1, [])] + [(PENDING, 0, 0, -1, -1, [])] * 2)
    rows = [(RESOLVED, 0, 0, 0, -1, [] if j == 0 else [(j - 1, False)]) for j in range(300)]
    rows.append((PENDING, 0, 255, -1, -1, [(299, False)]))
    tb.add_workflow(3, -10, rows)
    for pol in ("fcfs", "srtf", "lpt"):
        check(tb.build(), pol)
    # many instances / types near the limits
    s = random_table(99, n_workflows=40, max_rows=30, n_types=64, inst_per_type=(0, 16), max_cap=4)
    check(s, "srtf")


def test_validation_parity():
    nalar = _nalar()
    cases = []
    s = c1(); s.edges[3] = 23; cases.append(s)
    s = c1(); s.f_pin[7] = 0; cases.append(s)
    s = c1(); s.f_executor[3] = -1; cases.append(s)
    s = c1(); s.f_state[4] = 9; cases.append(s)
    s = c1(); s.f_type[11] = 5; cases.append(s)
    s = c2(1, n_workflows=30); s.edges[-1] = 5; cases.append(s)
    s = c2(1, n_workflows=30); s.edges[40] = 40; s.edges[100] = 3; cases.append(s)
    for s in cases:
        rc, row = oracle_validate(s)
        ctx = nalar.Context.for_snapshot(s)
        with pytest.raises(nalar.NalarError) as ei:
            ctx.upload(s)
        assert ei.value.code == nalar.NALAR_E_INVAL and ei.value.err_row == row
        with pytest.raises(nalar.NalarError) as ei:
            ctx.epoch("srtf")                  # no valid upload -> E_STATE
        assert ei.value.code == nalar.NALAR_E_STATE
        ctx.close()
    s = c2(1, n_workflows=30); s.wf_id[3] = s.wf_id[2]
    ctx = nalar.Context.for_snapshot(s)
    with pytest.raises(nalar.NalarError) as ei:
        ctx.upload(s)
    assert ei.value.err_row == -1
    big = c2(1, n_workflows=30)
    small = nalar.Context(10, 10, 2, 16, 4)
    with pytest.raises(nalar.NalarError) as ei:
        small.upload(big)
    assert ei.value.code == nalar.NALAR_E_NOMEM


# ---------------------------------------------------------------------------
# multi-GPU sharding on one GPU: G contexts, caller-side sum of the exchange
# buffers (the kernels all run on the GPU; only the allreduce is emulated)
# ---------------------------------------------------------------------------
class _CAI:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False),
                                         "version": 3}


def emulate_sharded(s, G, policy="srtf"):
    import torch
    nalar = _nalar()
    from paper_2601_05109_b200.sharding import shard_bounds
    bounds = shard_bounds(s.wf_fut_off, G)
    ctxs = []
    for k, (w0, w1) in enumerate(bounds):
        sh = s.slice_workflows(w0, w1)
        ctx = nalar.Context.for_snapshot(s, world=G, rank=k, collective=nalar.NALAR_COLL_EXTERNAL)
        ctx.upload(sh)
        ctx.begin(policy)
        ctxs.append((ctx, sh))
    torch.cuda.synchronize()
    bufs = []
    for ctx, _ in ctxs:
        p, n = ctx.exchange_buffer()
        bufs.append(torch.as_tensor(_CAI(p, n), device="cuda"))
    total = torch.stack([b.to(torch.int64) for b in bufs]).sum(0).to(torch.int32)
    for b in bufs:
        b.copy_(total)
    torch.cuda.synchronize()
    outs = []
    for ctx, sh in ctxs:
        ctx.finish()
        outs.append((ctx.fetch(), sh))
        ctx.close()
    return outs


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("which", ["c2", "c4", "rand"])
def test_sharded_equals_single(G, which):
    s = {"c2": lambda: c2(2), "c4": lambda: c4(3),
         "rand": lambda: random_table(77, n_workflows=40, max_rows=25, n_types=3,
                                      inst_per_type=(1, 3), max_cap=4)}[which]()
    o = oracle_epoch(s, "srtf")
    outs = emulate_sharded(s, G)
    for k in ("status", "level", "depth", "instance", "new_pin"):
        got = np.concatenate([g[k] for g, _ in outs])
        assert np.array_equal(got, o[k]), (k, G)
    assert np.array_equal(np.concatenate([g["wf_agg"] for g, _ in outs]), o["wf_agg"])
    for k in ("kv_hint", "kv_level", "kv_home"):
        assert np.array_equal(np.concatenate([g[k] for g, _ in outs]), o[k]), (k, G)
    for g, sh in outs:
        for k in ("i_load", "i_spare", "i_assigned"):
            assert np.array_equal(g[k], o[k]), (k, G)
        r0, r1 = sh.global_row_base, sh.global_row_base + sh.n_futures
        m = (o["assign_row"] >= r0) & (o["assign_row"] < r1)
        assert np.array_equal(g["assign_row"].astype(np.int64), o["assign_row"][m].astype(np.int64) - r0)
        assert np.array_equal(g["assign_inst"], o["assign_inst"][m])


def test_nccl_collective_in_graph_single_rank():
    """The library-owned NCCL communicator and the in-graph allreduce of the
    exchange buffer (world = 1: a one-rank communicator; the sum is the identity)."""
    import os
    os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")      # single-node bootstrap over loopback
    nalar = _nalar()
    uid = nalar.nalar_nccl_unique_id()
    for s in (c2(3), c4(1)):
        ctx = nalar.Context.for_snapshot(s, world=1, rank=0, collective=nalar.NALAR_COLL_NCCL,
                                         nccl_id=uid, flags=nalar.NALAR_F_TIMING)
        ctx.upload(s)
        for _ in range(3):                      # graph captured on the repeat, then replayed
            ctx.epoch("srtf")
        assert_same(s, oracle_epoch(s, "srtf"), ctx.fetch(), "nccl")
        assert ctx.stats().coll_us > 0
        ctx.close()
