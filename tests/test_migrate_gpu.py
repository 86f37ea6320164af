"""NEXT-1 HoL migration on the GPU (K1 candidates + K5 greedy) against oracle
O11, bit-exact: the destination of every migrated future, per-instance counts."""
import numpy as np
import pytest

from nalar_gen import c2, c4, hol_table, random_table, with_hol_inputs
from oracle import oracle_epoch

pytestmark = pytest.mark.gpu


def _nalar():
    from paper_2601_05109_b200 import nalar
    return nalar


def run(s, prm, policy="srtf", epochs=3, flags=0):
    nalar = _nalar()
    ctx = nalar.Context.for_snapshot(s, flags=flags)
    ctx.set_policy_params(migrate=True, theta_wait=prm["theta_wait"], theta_head=prm["theta_head"],
                          delta=prm["delta"])
    ctx.upload(s)
    outs = []
    for _ in range(epochs):               # direct launch, then graph capture + replay
        ctx.epoch(policy)
        outs.append(ctx.fetch())
    ctx.close()
    return outs


def check(s, prm, policy="srtf", **kw):
    o = oracle_epoch(s, policy, migrate={"f_age": s.f_age, "i_head_rem": s.i_head_rem, **prm})
    for g in run(s, prm, policy, **kw):
        assert np.array_equal(g["migrate_to"], o["migrate_to"]), np.nonzero(g["migrate_to"] != o["migrate_to"])
        assert np.array_equal(g["i_mig_in"], o["i_mig_in"]) and np.array_equal(g["i_mig_out"], o["i_mig_out"])
        assert g["n_migrated"] == o["n_migrated"]
        assert np.array_equal(g["status"], o["status"]) and np.array_equal(g["assign_row"], o["assign_row"])
    return o


@pytest.mark.parametrize("seed", range(80))
def test_hol_tables(seed):
    s = hol_table(seed, n_workflows=10 + seed % 40, n_types=1 + seed % 4, inst_per_type=1 + seed % 6)
    prm = {"theta_wait": seed % 12, "theta_head": (seed * 7) % 15, "delta": seed % 4}
    check(s, prm, ["fcfs", "srtf", "lpt"][seed % 3])


def test_hol_moves_happen():
    moved = 0
    for seed in range(20):
        s = hol_table(seed, n_workflows=60)
        moved += check(s, {"theta_wait": 5, "theta_head": 5, "delta": 1})["n_migrated"]
    assert moved > 50


@pytest.mark.parametrize("seed", range(20))
def test_hol_many_candidates_windows(seed):
    """More candidates per type than one placement window / warp batch."""
    s = hol_table(1000 + seed, n_workflows=2500, n_types=1 + seed % 2, inst_per_type=8, max_rows=3)
    check(s, {"theta_wait": 2, "theta_head": 5 + seed % 5, "delta": seed % 3}, epochs=1)


@pytest.mark.parametrize("mk", [lambda: c2(1), c4])
def test_hol_full_size(mk):
    s = with_hol_inputs(mk())
    check(s, {"theta_wait": 50, "theta_head": 50, "delta": 2})
    check(s, {"theta_wait": 10, "theta_head": 50, "delta": 0})


def test_hol_unstaged_and_no_inputs():
    nalar = _nalar()
    s = hol_table(5, n_workflows=50)
    check(s, {"theta_wait": 4, "theta_head": 4, "delta": 1}, flags=nalar.NALAR_F_FORCE_UNSTAGED)
    # migration on but no inputs uploaded -> nothing moves
    t = s.copy()
    t.f_age = None
    t.i_head_rem = None
    g = run(t, {"theta_wait": 0, "theta_head": 0, "delta": 0}, epochs=1)[0]
    assert g["n_migrated"] == 0 and (g["migrate_to"] == -1).all()


# ---- world > 1 (NEXT-1 across ranks): the candidates of every rank travel in
# the epoch's one exchange (list regions); every rank runs the same greedy -----

def _sharded_mig(s, G, prm, policy="srtf", collective="external", epochs=2):
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
        ctx.set_policy_params(migrate=True, theta_wait=prm["theta_wait"], theta_head=prm["theta_head"],
                              delta=prm["delta"])
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


def _check_sharded(s, G, prm, policy="srtf", **kw):
    o = oracle_epoch(s, policy, migrate={"f_age": s.f_age, "i_head_rem": s.i_head_rem, **prm})
    for outs in _sharded_mig(s, G, prm, policy, **kw):
        got = np.concatenate([g["migrate_to"] for g, _ in outs])
        assert np.array_equal(got, o["migrate_to"]), (G, np.nonzero(got != o["migrate_to"]))
        for g, _ in outs:
            assert np.array_equal(g["i_mig_in"], o["i_mig_in"]) and np.array_equal(g["i_mig_out"], o["i_mig_out"])
            assert g["n_migrated"] == o["n_migrated"]
        st = np.concatenate([g["status"] for g, _ in outs])
        assert np.array_equal(st, o["status"])
    return o


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("seed", range(6))
def test_hol_sharded_external(G, seed):
    s = hol_table(300 + seed, n_workflows=30 + 7 * seed, n_types=1 + seed % 3, inst_per_type=2 + seed % 5)
    prm = {"theta_wait": seed % 6, "theta_head": 3 + seed % 7, "delta": seed % 3}
    _check_sharded(s, G, prm, ["fcfs", "srtf", "lpt"][seed % 3])


@pytest.mark.parametrize("G", [2, 4, 8])
def test_hol_sharded_c4(G):
    s = with_hol_inputs(c4(2))
    o = _check_sharded(s, G, {"theta_wait": 0, "theta_head": 10, "delta": 0})
    assert o["n_migrated"] > 0


@pytest.mark.parametrize("G", [2, 3, 4])
def test_hol_sharded_peer(G):
    s = with_hol_inputs(c2(3))
    _check_sharded(s, G, {"theta_wait": 10, "theta_head": 50, "delta": 1}, collective="peer", epochs=3)
    s = hol_table(77, n_workflows=60, n_types=2, inst_per_type=5)
    _check_sharded(s, G, {"theta_wait": 3, "theta_head": 5, "delta": 1}, collective="peer", epochs=3)


def test_hol_sharded_list_overflow_is_reported():
    """More candidates on a rank than its list region holds: E_NOTIMPL at the
    fetch on every rank, never a partial answer."""
    nalar = _nalar()
    s = hol_table(5, n_workflows=40000, n_types=1, inst_per_type=8, max_rows=3)
    prm = {"theta_wait": 0, "theta_head": 0, "delta": 0}
    with pytest.raises(nalar.NalarError) as e:
        _check_sharded(s, 2, prm, epochs=1)
    assert e.value.code == nalar.NALAR_E_NOTIMPL
