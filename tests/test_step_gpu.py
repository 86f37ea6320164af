"""nalar_step (upload + epoch + fetch with one synchronisation) against the
oracle and against the three split calls; invalid tables through the step
(validation verdict read after the fetch, the epoch kernels skipping the
table on the device)."""
import numpy as np
import pytest

from nalar_gen import Snapshot, c1, c2, c4, random_table, swe_table
from oracle import oracle_epoch

pytestmark = pytest.mark.gpu

KEYS = ("status", "level", "depth", "instance", "new_pin", "wf_agg", "i_load", "i_spare",
        "i_assigned", "assign_row", "assign_inst", "kv_hint", "kv_level", "kv_home")


def _nalar():
    from paper_2601_05109_b200 import nalar
    return nalar


def same(o, g, tag):
    for k in KEYS:
        assert np.array_equal(np.asarray(o[k]), np.asarray(g[k])), (tag, k)


def pinned_like(a, keep):
    import torch
    t = torch.empty(max(a.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    keep.append(t)
    v = t.numpy()[:a.nbytes].view(a.dtype).reshape(a.shape)
    v[...] = a
    return v


@pytest.mark.parametrize("mk", [c1, lambda: c2(1), lambda: swe_table(5000, seed=3), c4,
                                lambda: random_table(9, n_workflows=7, max_rows=30, consistent=True)])
@pytest.mark.parametrize("policy", ["srtf", "lpt", "fcfs"])
def test_step_matches_oracle(mk, policy):
    nalar = _nalar()
    s = mk()
    o = oracle_epoch(s, policy)
    ctx = nalar.Context.for_snapshot(s)
    for _ in range(3):                       # direct launch, graph capture, replay
        same(o, ctx.step(s, policy), f"{s.name} {policy}")
    ctx.close()


def test_step_pinned_in_and_out():
    """The configuration bench.py's e2e leg times: pinned inputs and outputs."""
    nalar = _nalar()
    keep = []
    s = c4()
    o = oracle_epoch(s, "srtf")
    sp = Snapshot(global_row_base=0, name="pinned", **{k: pinned_like(v, keep) for k, v in s.arrays().items()})
    ctx = nalar.Context.for_snapshot(s)
    out = ctx.output_buffers(("status", "instance", "assign"),
                             alloc=lambda n, dt: pinned_like(np.zeros(n, dt), keep), like=s)
    for _ in range(3):
        g = ctx.step(sp, "srtf", ("status", "instance", "assign"), out=out)
        for k in ("status", "instance", "assign_row", "assign_inst"):
            assert np.array_equal(np.asarray(o[k]), np.asarray(g[k])), k
    ctx.close()


def _bad_edge(s, row, to):
    arrs = s.arrays()
    edges = arrs["edges"].copy()
    edges[int(arrs["f_edge_off"][row])] = to
    return Snapshot(global_row_base=0, name="bad", **{**arrs, "edges": edges})


def test_step_invalid_table_reports_row_then_recovers():
    nalar = _nalar()
    s = swe_table(6000, seed=4)
    # a forward edge from some row with edges: the smallest offending row is reported
    rows = np.nonzero(np.diff(s.f_edge_off.astype(np.int64)) > 0)[0]
    r = int(rows[len(rows) // 2])
    bad = _bad_edge(s, r, r + 1)
    ctx = nalar.Context.for_snapshot(s)
    with pytest.raises(nalar.NalarError) as e:
        ctx.upload(bad)
    want = e.value.err_row
    assert want == r
    for _ in range(2):
        with pytest.raises(nalar.NalarError) as e:
            ctx.step(bad, "srtf")
        assert e.value.code == nalar.NALAR_E_INVAL and e.value.err_row == want
        with pytest.raises(nalar.NalarError) as e:
            ctx.fetch()                      # the failed step left nothing to fetch
        assert e.value.code == nalar.NALAR_E_STATE
    # a valid table through the same context afterwards (graph replays included)
    o = oracle_epoch(s, "srtf")
    for _ in range(3):
        same(o, ctx.step(s, "srtf"), "after invalid")
    ctx.close()


def test_step_structurally_invalid_offsets_do_not_crash():
    """Non-monotone edge offsets (the K1 block tables computed from them are
    garbage): the device skips the epoch, the step reports E_INVAL."""
    nalar = _nalar()
    s = swe_table(4000, seed=8)
    arrs = s.arrays()
    eo = arrs["f_edge_off"].copy()
    mid = len(eo) // 2
    eo[mid], eo[mid + 1] = eo[mid + 1] + 5, eo[mid]
    bad = Snapshot(global_row_base=0, name="badoff", **{**arrs, "f_edge_off": eo})
    ctx = nalar.Context.for_snapshot(s)
    with pytest.raises(nalar.NalarError) as e:
        ctx.step(bad, "srtf")
    assert e.value.code == nalar.NALAR_E_INVAL
    same(oracle_epoch(s, "lpt"), ctx.step(s, "lpt"), "after structural")
    ctx.close()


def test_step_with_next_rows():
    nalar = _nalar()
    s = c4()
    o = oracle_epoch(s, "srtf", reassign={"u_hi_pct": 80, "u_lo_pct": 30})
    ctx = nalar.Context.for_snapshot(s)
    ctx.set_policy_params(reassign=True, u_hi_pct=80, u_lo_pct=30)
    for _ in range(2):
        g = ctx.step(s, "srtf")
        same(o, g, "reassign")
        assert np.array_equal(g["ra_kill"], o["ra_kill"]) and np.array_equal(g["ra_prov"], o["ra_prov"])
    ctx.close()


# ---- the streamed step (pinned per-row arrays: K1 stages them from host memory,
# validates them in shared memory and writes the device copy) -------------------

def _pinned_snapshot(s, keep, name="pinned"):
    return Snapshot(global_row_base=0, name=name, **{k: pinned_like(v, keep) for k, v in s.arrays().items()})


@pytest.mark.parametrize("mk", [c1, lambda: c2(1), lambda: swe_table(5000, seed=3), c4,
                                lambda: random_table(9, n_workflows=7, max_rows=30, consistent=True),
                                lambda: random_table(21, n_workflows=40, max_rows=70)])
@pytest.mark.parametrize("policy", ["srtf", "lpt", "fcfs"])
def test_streamed_step_matches_oracle(mk, policy):
    nalar = _nalar()
    keep = []
    s = mk()
    o = oracle_epoch(s, policy)
    sp = _pinned_snapshot(s, keep)
    ctx = nalar.Context.for_snapshot(s)
    for _ in range(3):                       # direct launch, graph capture, replay
        same(o, ctx.step(sp, policy), f"{s.name} {policy}")
        assert ctx.last_step_streamed()
    ctx.close()


def test_streamed_step_writes_the_device_table():
    """Split calls after a streamed step run on the device copy the sweep wrote."""
    nalar = _nalar()
    keep = []
    s = c4()
    sp = _pinned_snapshot(s, keep)
    ctx = nalar.Context.for_snapshot(s)
    same(oracle_epoch(s, "srtf"), ctx.step(sp, "srtf"), "streamed")
    assert ctx.last_step_streamed()
    for pol in ("lpt", "fcfs"):
        ctx.epoch(pol)
        same(oracle_epoch(s, pol), ctx.fetch(), f"split {pol} after streamed")
    ctx.close()


def test_streamed_step_invalid_rows_and_offsets():
    nalar = _nalar()
    keep = []
    s = swe_table(6000, seed=4)
    rows = np.nonzero(np.diff(s.f_edge_off.astype(np.int64)) > 0)[0]
    r = int(rows[len(rows) // 3])
    bad = _pinned_snapshot(_bad_edge(s, r, r + 1), keep, "bad")
    ctx = nalar.Context.for_snapshot(s)
    for _ in range(2):
        with pytest.raises(nalar.NalarError) as e:
            ctx.step(bad, "srtf")
        assert e.value.code == nalar.NALAR_E_INVAL and e.value.err_row == r
        assert ctx.last_step_streamed()
    # an edge to a row of another workflow and a pin of the wrong type: the
    # smallest offending row over all blocks is reported, as K0 does
    arrs = s.arrays()
    pin = arrs["f_pin"].copy()
    it = arrs["i_type"]
    r2 = len(pin) - 7
    pin[r2] = int(np.nonzero(it != arrs["f_type"][r2])[0][0])
    edges = arrs["edges"].copy()
    r3 = int(rows[-5])
    edges[int(arrs["f_edge_off"][r3])] = 0        # row 0 is in the first workflow
    two = _pinned_snapshot(Snapshot(global_row_base=0, name="two", **{**arrs, "f_pin": pin, "edges": edges}), keep)
    with pytest.raises(nalar.NalarError) as e:
        ctx.upload(Snapshot(global_row_base=0, name="two", **{**arrs, "f_pin": pin, "edges": edges}))
    want = e.value.err_row
    with pytest.raises(nalar.NalarError) as e:
        ctx.step(two, "srtf")
    assert e.value.err_row == want == min(r2, r3)
    # non-monotone offsets
    eo = arrs["f_edge_off"].copy()
    mid = len(eo) // 2
    eo[mid], eo[mid + 1] = eo[mid + 1] + 5, eo[mid]
    badoff = _pinned_snapshot(Snapshot(global_row_base=0, name="badoff", **{**arrs, "f_edge_off": eo}), keep)
    with pytest.raises(nalar.NalarError) as e:
        ctx.step(badoff, "srtf")
    assert e.value.code == nalar.NALAR_E_INVAL
    # recovery: valid streamed steps, then split calls on the written table
    good = _pinned_snapshot(s, keep)
    for _ in range(3):
        same(oracle_epoch(s, "srtf"), ctx.step(good, "srtf"), "after invalid")
        assert ctx.last_step_streamed()
    ctx.epoch("lpt")
    same(oracle_epoch(s, "lpt"), ctx.fetch(), "split after recovery")
    ctx.close()


def test_streamed_step_falls_back_when_a_block_is_unstaged():
    nalar = _nalar()
    keep = []
    s = swe_table(3000, seed=6)
    sp = _pinned_snapshot(s, keep)
    ctx = nalar.Context.for_snapshot(s, flags=nalar.NALAR_F_FORCE_UNSTAGED)
    for _ in range(2):
        same(oracle_epoch(s, "srtf"), ctx.step(sp, "srtf"), "unstaged")
        assert not ctx.last_step_streamed()
    ctx.close()


def test_streamed_step_off_for_pageable_and_next_rows():
    nalar = _nalar()
    keep = []
    s = swe_table(4000, seed=2)
    ctx = nalar.Context.for_snapshot(s)
    same(oracle_epoch(s, "srtf"), ctx.step(s, "srtf"), "pageable")
    assert not ctx.last_step_streamed()
    # reassignment (in K4) streams; batch coalescing (K6) keeps the plain path
    sp = _pinned_snapshot(s, keep)
    ctx.set_policy_params(reassign=True, u_hi_pct=80, u_lo_pct=30)
    o = oracle_epoch(s, "srtf", reassign={"u_hi_pct": 80, "u_lo_pct": 30})
    g = ctx.step(sp, "srtf")
    same(o, g, "streamed reassign")
    assert ctx.last_step_streamed()
    assert np.array_equal(g["ra_kill"], o["ra_kill"]) and np.array_equal(g["ra_prov"], o["ra_prov"])
    mb = np.full(s.n_types, 1, np.uint16)
    mb[[t for t in range(s.n_types) if s.t_affinity[t] == 0][:2]] = 3
    ctx.set_policy_params(t_max_batch=mb, n_types=s.n_types)
    ob = oracle_epoch(s, "srtf", batch={"t_max_batch": mb, "f_method": s.f_method})
    g = ctx.step(sp, "srtf")
    same(ob, g, "batch")
    assert np.array_equal(g["batch_head"], ob["batch_head"])
    assert not ctx.last_step_streamed()
    ctx.close()


# ---- streamed outputs: with every per-row output pinned, K1 / K4 write them
# straight to the caller's memory during the epoch (the fetch skips them) ----

@pytest.mark.parametrize("mk", [c1, lambda: c2(1), c4, lambda: random_table(33, n_workflows=30, max_rows=40),
                                lambda: swe_table(20000, seed=5)])
@pytest.mark.parametrize("policy", ["srtf", "lpt"])
def test_streamed_outputs_all_fields(mk, policy):
    nalar = _nalar()
    keep = []
    s = mk()
    o = oracle_epoch(s, policy)
    sp = _pinned_snapshot(s, keep)
    ctx = nalar.Context.for_snapshot(s)
    out = ctx.output_buffers(("status", "level", "depth", "instance", "new_pin", "wf_agg", "i_load", "i_spare",
                              "i_assigned", "assign", "kv"),
                             alloc=lambda n, dt: pinned_like(np.zeros(n, dt), keep), like=s)
    for k in ("status", "level", "depth", "instance", "new_pin"):
        out[k][...] = 0x5A                     # poison: every row must be written
    for _ in range(3):                         # direct launch, graph capture, replay
        g = ctx.step(sp, policy, out=out)
        same(o, g, f"{s.name} {policy} streamed outputs")
    # a split fetch afterwards (the plain copy path) agrees
    ctx.epoch(policy)
    same(o, ctx.fetch(), "split after streamed outputs")
    ctx.close()


def test_streamed_outputs_pageable_inputs_and_reassign():
    """Pageable inputs (plain upload) with pinned outputs still stream the outputs."""
    nalar = _nalar()
    keep = []
    s = c4(2)
    prm = {"u_hi_pct": 80, "u_lo_pct": 30}
    o = oracle_epoch(s, "srtf", reassign=prm)
    ctx = nalar.Context.for_snapshot(s)
    ctx.set_policy_params(reassign=True, **prm)
    out = ctx.output_buffers(("status", "level", "depth", "instance", "new_pin", "assign", "reassign"),
                             alloc=lambda n, dt: pinned_like(np.zeros(n, dt), keep), like=s)
    for _ in range(2):
        g = ctx.step(s, "srtf", out=out)
        for k in ("status", "level", "depth", "instance", "new_pin", "assign_row", "assign_inst"):
            assert np.array_equal(np.asarray(g[k]), np.asarray(o[k])), k
        assert np.array_equal(g["ra_kill"], o["ra_kill"])
    ctx.close()
