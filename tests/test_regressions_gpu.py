"""Regression tests for the round-1 advisor findings, on the GPU,
against the oracle where a result is compared.

- the epoch-graph cache must not replay a graph captured for other per-upload
  inputs (HoL inputs present or not, methods present or not, affinities);
- a delta clears the per-upload batch methods (rows moved);
- fetch / step must refuse caller buffers shorter than the table (E_SIZE);
- a failed peer exchange is sticky and spreads to the peers, and a reconnect
  recovers;
- an empty table uploaded after an invalid one is valid (the device verdict
  word is cleared).
"""
import numpy as np
import pytest

from nalar_gen import AFF_NONE, c1, c2, random_table, swe_table, with_hol_inputs
from oracle import oracle_epoch

pytestmark = pytest.mark.gpu


def _nalar():
    from paper_2601_05109_b200 import nalar
    return nalar


def _same(o, g, keys=("status", "level", "instance", "new_pin", "assign_row", "assign_inst")):
    for k in keys:
        assert np.array_equal(np.asarray(o[k]), np.asarray(g[k])), k


def test_graph_key_hol_inputs_dropped():
    """Same shape, HoL inputs present then absent: the replay must not keep the
    migration kernel (stale migrate_to)."""
    nalar = _nalar()
    base = swe_table(6000, seed=5)
    s_mig = with_hol_inputs(base, seed=5)
    prm = {"theta_wait": 2, "theta_head": 2, "delta": 1}
    ctx = nalar.Context.for_snapshot(s_mig)
    ctx.set_policy_params(migrate=True, **prm)
    ctx.upload(s_mig)
    for _ in range(3):
        ctx.epoch("srtf")
    g = ctx.fetch()
    o = oracle_epoch(s_mig, "srtf", migrate={"f_age": s_mig.f_age, "i_head_rem": s_mig.i_head_rem, **prm})
    assert o["n_migrated"] > 0 and np.array_equal(g["migrate_to"], o["migrate_to"])
    ctx.upload(base)                                  # no f_age / i_head_rem: nothing migrates
    for _ in range(3):
        ctx.epoch("srtf")
        g = ctx.fetch()
        assert g["n_migrated"] == 0 and (g["migrate_to"] == -1).all()
        _same(oracle_epoch(base, "srtf"), g)
    ctx.upload(s_mig)                                 # and back
    for _ in range(2):
        ctx.epoch("srtf")
    g = ctx.fetch()
    assert np.array_equal(g["migrate_to"], o["migrate_to"])
    ctx.close()


def test_graph_key_methods_added_and_dropped():
    nalar = _nalar()
    s = random_table(3, n_workflows=40, max_rows=20, n_types=3, inst_per_type=(1, 3), max_cap=8, p_pin=0.2)
    s.t_affinity[:] = AFF_NONE
    mb = np.array([3, 2, 4])
    with_m = s.copy()
    with_m.f_method = np.random.default_rng(1).integers(0, 3, s.n_futures).astype(np.uint8)
    ctx = nalar.Context.for_snapshot(s)
    ctx.set_policy_params(t_max_batch=mb, n_types=s.n_types)
    for snap in (s, with_m, s, with_m):
        ctx.upload(snap)
        o = oracle_epoch(snap, "srtf", batch={"t_max_batch": mb, "f_method": snap.f_method})
        for _ in range(3):                            # direct, capture, replay
            ctx.epoch("srtf")
            g = ctx.fetch()
            assert np.array_equal(g["batch_head"], o["batch_head"])
            assert g["n_batches"] == o["n_batches"]
    ctx.close()


def test_graph_key_affinity_change_rechecks():
    """A re-upload that gives a batchable type managed state must be rejected
    even when the same-shape epoch graph is cached."""
    nalar = _nalar()
    s = random_table(4, n_workflows=30, max_rows=15, n_types=2, inst_per_type=(1, 3), max_cap=6)
    s.t_affinity[:] = AFF_NONE
    ctx = nalar.Context.for_snapshot(s)
    ctx.set_policy_params(t_max_batch=np.array([2, 2]), n_types=2)
    ctx.upload(s)
    for _ in range(3):
        ctx.epoch("srtf")
    bad = s.copy()
    bad.t_affinity[:] = 1                            # SESSION
    bad.f_pin[:] = -1
    ctx.upload(bad)
    with pytest.raises(nalar.NalarError) as e:
        ctx.epoch("srtf")
    assert e.value.code == nalar.NALAR_E_INVAL
    ctx.close()


def test_delta_clears_methods():
    from tests.test_delta_cpu import apply_delta_ref
    from tests.test_delta_gpu import _manual_delta
    nalar = _nalar()
    rng = np.random.default_rng(9)
    s = random_table(9, n_workflows=60, max_rows=15, n_types=3, inst_per_type=(1, 4), max_cap=5, p_pin=0.2)
    s.t_affinity[:] = AFF_NONE
    s.f_method = rng.integers(0, 3, s.n_futures).astype(np.uint8)
    mb = np.array([2, 3, 2])
    ctx = nalar.Context(120000, 240000, 2000, 64, 8)
    ctx.set_policy_params(t_max_batch=mb, n_types=s.n_types)
    ctx.upload(s)
    o = oracle_epoch(s, "srtf", batch={"t_max_batch": mb, "f_method": s.f_method})
    ctx.epoch("srtf")
    g = ctx.fetch()
    assert np.array_equal(g["batch_head"], o["batch_head"])
    d = _manual_delta(s, rng, o)
    s2 = apply_delta_ref(s, o["assign_row"], o["assign_inst"], d)
    d.n_futures_after, d.n_workflows_after = s2.n_futures, s2.n_workflows
    ctx.apply_delta(d)
    o2 = oracle_epoch(s2, "srtf", batch={"t_max_batch": mb, "f_method": None})
    ctx.epoch("srtf")
    g2 = ctx.fetch()
    assert np.array_equal(g2["batch_head"], o2["batch_head"]) and g2["n_batches"] == o2["n_batches"]
    ctx.close()


@pytest.mark.parametrize("field", ["status", "depth", "wf_agg", "i_load"])
def test_short_output_buffers_rejected(field):
    nalar = _nalar()
    small, big = swe_table(1000, seed=1), swe_table(3000, seed=2)
    ctx = nalar.Context.for_snapshot(big)
    ctx.upload(big)
    ctx.epoch("srtf")
    out = ctx.output_buffers(like=big)
    out[field] = out[field][: out[field].size // 2].copy()
    with pytest.raises(nalar.NalarError) as e:
        ctx.fetch(out=out)
    assert e.value.code == nalar.NALAR_E_SIZE
    # buffers sized for a smaller table, reused for a bigger one
    out = ctx.output_buffers(like=small)
    with pytest.raises(nalar.NalarError) as e:
        ctx.step(big, out=out)
    assert e.value.code == nalar.NALAR_E_SIZE
    ctx.close()


def test_peer_failure_is_sticky_and_reconnect_recovers():
    import torch
    from paper_2601_05109_b200.sharding import connect_local, shard_bounds
    nalar = _nalar()
    s = c2(2, n_workflows=300)
    G = 2
    streams = [torch.cuda.Stream() for _ in range(G)]
    ctxs, shards = [], []
    for k, (w0, w1) in enumerate(shard_bounds(s.wf_fut_off, G)):
        ctxs.append(nalar.Context.for_snapshot(s, world=G, rank=k, collective=nalar.NALAR_COLL_PEER,
                                               stream=streams[k].cuda_stream, flags=nalar.NALAR_F_NO_GRAPH))
        shards.append(s.slice_workflows(w0, w1))
    connect_local(ctxs)
    for c, sh in zip(ctxs, shards):
        c.upload(sh)
    o = oracle_epoch(s, "srtf")
    # rank 1 skips an epoch: rank 0 times out (5 s) and fails
    ctxs[0].epoch("srtf")
    with pytest.raises(nalar.NalarError) as e:
        ctxs[0].fetch()
    assert e.value.code == nalar.NALAR_E_COMM
    # rank 1's epoch would pair with rank 0's stale slot: it must fail at once
    ctxs[1].epoch("srtf")
    with pytest.raises(nalar.NalarError) as e:
        ctxs[1].fetch()
    assert e.value.code == nalar.NALAR_E_COMM
    # both are sticky-failed
    for c in ctxs:
        with pytest.raises(nalar.NalarError) as e:
            c.epoch("srtf")
        assert e.value.code == nalar.NALAR_E_COMM
    # reconnect: exact results again
    connect_local(ctxs)
    for _ in range(2):
        for c in ctxs:
            c.epoch("srtf")
        outs = [c.fetch() for c in ctxs]
    for k in ("status", "level", "instance"):
        assert np.array_equal(np.concatenate([g[k] for g in outs]), o[k]), k
    for c in ctxs:
        c.close()


def test_empty_table_after_invalid_upload():
    nalar = _nalar()
    s = c1()
    ctx = nalar.Context.for_snapshot(s)
    bad = s.copy()
    bad.edges[3] = 23
    with pytest.raises(nalar.NalarError):
        ctx.step(bad)
    empty = s.slice_workflows(0, 0)
    g = ctx.step(empty)
    assert g["n_assigned"] == 0
    assert np.array_equal(g["i_load"], s.i_base_load) and np.array_equal(g["i_assigned"], np.zeros(s.n_instances))
    o = oracle_epoch(empty, "srtf")
    assert np.array_equal(g["i_spare"], o["i_spare"])
    ctx.close()
