"""NEXT-4 batch coalescing on the GPU (K6) against oracle O12, bit-exact."""
import numpy as np
import pytest

from nalar_gen import AFF_NONE, c2, c4, random_table
from oracle import oracle_epoch

pytestmark = pytest.mark.gpu


def _nalar():
    from paper_2601_05109_b200 import nalar
    return nalar


def check(s, mb, policy="srtf", epochs=3, flags=0):
    nalar = _nalar()
    o = oracle_epoch(s, policy, batch={"t_max_batch": mb, "f_method": s.f_method})
    ctx = nalar.Context.for_snapshot(s, flags=flags)
    ctx.set_policy_params(t_max_batch=mb, n_types=s.n_types)
    ctx.upload(s)
    for _ in range(epochs):
        ctx.epoch(policy)
        g = ctx.fetch()
        assert np.array_equal(g["batch_head"], o["batch_head"]), np.nonzero(g["batch_head"] != o["batch_head"])
        assert g["n_batches"] == o["n_batches"]
        assert np.array_equal(g["assign_row"], o["assign_row"])
    ctx.close()
    return o


@pytest.mark.parametrize("seed", range(60))
def test_batch_random(seed):
    rng = np.random.default_rng(seed)
    s = random_table(seed, n_workflows=3 + seed % 8, max_rows=4 + seed % 25, n_types=1 + seed % 3,
                     inst_per_type=(1, 3), consistent=seed % 2 == 0, max_cap=2 + seed % 9, p_pin=0.3)
    s.t_affinity[:] = AFF_NONE
    s.f_method = rng.integers(0, 1 + seed % 4, s.n_futures)
    check(s, rng.integers(0, 5, s.n_types), ["fcfs", "srtf", "lpt"][seed % 3])


@pytest.mark.parametrize("mk", [lambda: c2(1), c4])
def test_batch_full_size(mk):
    s = mk()
    rng = np.random.default_rng(3)
    s.f_method = rng.integers(0, 3, s.n_futures)
    mb = np.where(s.t_affinity == AFF_NONE, 4, 0)
    o = check(s, mb)
    assert o["n_batches"] > 0


def test_batch_managed_state_rejected_and_off():
    nalar = _nalar()
    s = c4()
    ctx = nalar.Context.for_snapshot(s)
    ctx.upload(s)
    ctx.set_policy_params(t_max_batch=np.full(8, 4), n_types=8)      # SESSION / STATEFUL types too
    with pytest.raises(nalar.NalarError):
        ctx.epoch("srtf")
    ctx.set_policy_params()
    ctx.epoch("srtf")
    g = ctx.fetch()
    assert g["n_batches"] == 0 and (g["batch_head"] == -1).all()
    ctx.close()


@pytest.mark.parametrize("unpin", [False, True])
def test_batch_long_sequences_fallback(unpin):
    """Instances receiving more futures than K6 stages in shared memory (1024
    per sequence): one instance per type takes all of its type's work, so its
    sequence (phase B, or phase A once every future is pinned to it) exceeds
    the staging and the global-memory merge runs -- the same batches."""
    from nalar_gen import swe_table
    s = swe_table(400000, seed=7)
    s.t_affinity[:] = AFF_NONE
    first = np.array([np.nonzero(s.i_type == t)[0][0] for t in range(s.n_types)])
    cap = np.zeros(s.n_instances, dtype=s.i_cap.dtype)
    cap[first] = 1000000
    s.i_cap[:] = cap
    s.i_base_load[:] = 0
    if unpin:
        s.f_pin[:] = np.where(s.f_state == 0, first[s.f_type], s.f_pin)
    rng = np.random.default_rng(5)
    s.f_method = rng.integers(0, 3, s.n_futures)
    o = check(s, np.full(s.n_types, 5), epochs=2)
    inst = o["instance"][o["status"] == 7]
    assert np.bincount(inst).max() > 1024


# ---- world > 1 (NEXT-4 across ranks): every rank's eligible futures of the
# batchable resources travel in the epoch's one exchange; every rank re-derives
# their admission and cuts every instance's batches (global rows) -------------

def _sharded_batch(s, G, mb, policy="srtf", collective="external", epochs=2):
    import torch
    from tests.test_parity_gpu import _CAI
    from paper_2601_05109_b200.sharding import connect_local, shard_bounds
    nalar = _nalar()
    coll = {"external": nalar.NALAR_COLL_EXTERNAL, "peer": nalar.NALAR_COLL_PEER}[collective]
    streams = [torch.cuda.Stream() for _ in range(G)] if collective == "peer" else [None] * G
    ctxs, shards = [], []
    for k, (w0, w1) in enumerate(shard_bounds(s.wf_fut_off, G)):
        kw = {"stream": streams[k].cuda_stream} if streams[k] is not None else {}
        ctx = nalar.Context.for_snapshot(s, world=G, rank=k, collective=coll, **kw)
        ctx.set_policy_params(t_max_batch=mb, n_types=s.n_types)
        ctxs.append(ctx)
        shards.append(s.slice_workflows(w0, w1))
    if collective == "peer":
        connect_local(ctxs)
    for c, sh in zip(ctxs, shards):
        c.upload(sh)
    outs = []
    for _ in range(epochs):
        if collective == "peer":
            for c in ctxs:
                c.epoch(policy)
        else:
            for c in ctxs:
                c.begin(policy)
            torch.cuda.synchronize()
            bufs = [torch.as_tensor(_CAI(*c.exchange_buffer()), device="cuda") for c in ctxs]
            total = torch.stack([b.to(torch.int64) for b in bufs]).sum(0).to(torch.int32)
            for b in bufs:
                b.copy_(total)
            torch.cuda.synchronize()
            for c in ctxs:
                c.finish()
        outs.append([(c.fetch(), sh) for c, sh in zip(ctxs, shards)])
    for c in ctxs:
        c.close()
    return outs


def _check_batch_sharded(s, G, mb, policy="srtf", **kw):
    o = oracle_epoch(s, policy, batch={"t_max_batch": mb, "f_method": s.f_method})
    for outs in _sharded_batch(s, G, mb, policy, **kw):
        got = np.concatenate([g["batch_head"] for g, _ in outs])
        assert np.array_equal(got, o["batch_head"]), (G, np.nonzero(got != o["batch_head"]))
        for g, _ in outs:
            assert g["n_batches"] == o["n_batches"]
    return o


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("seed", range(8))
def test_batch_sharded_external(G, seed):
    rng = np.random.default_rng(100 + seed)
    s = random_table(200 + seed, n_workflows=20 + 5 * seed, max_rows=6 + seed % 20, n_types=1 + seed % 3,
                     inst_per_type=(1, 3), consistent=seed % 2 == 0, max_cap=2 + seed % 9, p_pin=0.3)
    s.t_affinity[:] = AFF_NONE
    s.f_method = rng.integers(0, 1 + seed % 4, s.n_futures).astype(np.uint8)
    _check_batch_sharded(s, G, rng.integers(0, 5, s.n_types), ["fcfs", "srtf", "lpt"][seed % 3])


@pytest.mark.parametrize("G", [2, 4, 8])
def test_batch_sharded_c4(G):
    s = c4(2)
    s.f_method = np.random.default_rng(3).integers(0, 3, s.n_futures).astype(np.uint8)
    mb = np.where(s.t_affinity == AFF_NONE, 4, 0)
    o = _check_batch_sharded(s, G, mb)
    assert o["n_batches"] > 0


@pytest.mark.parametrize("G", [2, 3])
def test_batch_sharded_peer(G):
    s = c2(2)
    s.f_method = np.random.default_rng(5).integers(0, 2, s.n_futures).astype(np.uint8)
    mb = np.where(s.t_affinity == AFF_NONE, 3, 0)
    o = _check_batch_sharded(s, G, mb, collective="peer", epochs=3)
    assert o["n_batches"] > 0


def test_batch_and_migration_sharded_together():
    """Both list sections in one exchange."""
    import torch
    from tests.test_parity_gpu import _CAI
    from paper_2601_05109_b200.sharding import shard_bounds
    from nalar_gen import hol_table
    nalar = _nalar()
    s = hol_table(9, n_workflows=80, n_types=3, inst_per_type=4)
    s.t_affinity[:] = AFF_NONE
    s.f_method = np.random.default_rng(9).integers(0, 2, s.n_futures).astype(np.uint8)
    mb = np.full(s.n_types, 2)
    prm = {"theta_wait": 2, "theta_head": 4, "delta": 1}
    o = oracle_epoch(s, "srtf", batch={"t_max_batch": mb, "f_method": s.f_method},
                     migrate={"f_age": s.f_age, "i_head_rem": s.i_head_rem, **prm})
    G = 3
    ctxs, shards = [], []
    for k, (w0, w1) in enumerate(shard_bounds(s.wf_fut_off, G)):
        ctx = nalar.Context.for_snapshot(s, world=G, rank=k, collective=nalar.NALAR_COLL_EXTERNAL)
        ctx.set_policy_params(t_max_batch=mb, n_types=s.n_types, migrate=True, **prm)
        sh = s.slice_workflows(w0, w1)
        ctx.upload(sh)
        ctx.begin("srtf")
        ctxs.append(ctx)
        shards.append(sh)
    torch.cuda.synchronize()
    bufs = [torch.as_tensor(_CAI(*c.exchange_buffer()), device="cuda") for c in ctxs]
    total = torch.stack([b.to(torch.int64) for b in bufs]).sum(0).to(torch.int32)
    for b in bufs:
        b.copy_(total)
    torch.cuda.synchronize()
    outs = []
    for c in ctxs:
        c.finish()
        outs.append(c.fetch())
        c.close()
    assert np.array_equal(np.concatenate([g["batch_head"] for g in outs]), o["batch_head"])
    assert np.array_equal(np.concatenate([g["migrate_to"] for g in outs]), o["migrate_to"])
    assert all(g["n_batches"] == o["n_batches"] and g["n_migrated"] == o["n_migrated"] for g in outs)
