"""NEXT-2 resource reassignment on the GPU (K4 type blocks + last-block
pairing) against oracle O10, bit-exact, on one GPU and sharded."""
import numpy as np
import pytest

from nalar_gen import c2, c4, random_table
from oracle import oracle_epoch

pytestmark = pytest.mark.gpu


def _nalar():
    from paper_2601_05109_b200 import nalar
    return nalar


def run(s, prm, policy="srtf"):
    nalar = _nalar()
    ctx = nalar.Context.for_snapshot(s)
    ctx.set_policy_params(reassign=True, u_hi_pct=prm["u_hi_pct"], u_lo_pct=prm["u_lo_pct"],
                          t_min_inst=prm.get("t_min_inst"), t_max_inst=prm.get("t_max_inst"),
                          n_types=s.n_types)
    ctx.upload(s)
    outs = []
    for _ in range(3):                   # direct launch, then graph capture + replay
        ctx.epoch(policy)
        outs.append(ctx.fetch())
    ctx.close()
    return outs


def same(o, g):
    assert np.array_equal(g["t_busy"], o["t_busy"]), (g["t_busy"], o["t_busy"])
    assert np.array_equal(g["t_capsum"], o["t_cap"])
    assert np.array_equal(g["ra_kill"], o["ra_kill"]) and np.array_equal(g["ra_prov"], o["ra_prov"])
    assert np.array_equal(g["status"], o["status"]) and np.array_equal(g["assign_row"], o["assign_row"])


@pytest.mark.parametrize("seed", range(60))
def test_reassign_random(seed):
    rng = np.random.default_rng(seed)
    s = random_table(seed, n_workflows=2 + seed % 5, max_rows=4 + seed % 20, n_types=1 + seed % 5,
                     inst_per_type=(0, 1 + seed % 4), consistent=seed % 2 == 1, max_cap=1 + seed % 7,
                     max_base=seed % 9)
    T = s.n_types
    prm = {"t_min_inst": rng.integers(0, 3, T).tolist(), "t_max_inst": rng.integers(1, 6, T).tolist(),
           "u_hi_pct": int(rng.integers(30, 120))}
    prm["u_lo_pct"] = min(int(rng.integers(0, 50)), prm["u_hi_pct"])
    o = oracle_epoch(s, "srtf", reassign=prm)
    for g in run(s, prm):
        same(o, g)


@pytest.mark.parametrize("mk", [lambda: c2(1), c4])
def test_reassign_full_size(mk):
    s = mk()
    prm = {"u_hi_pct": 80, "u_lo_pct": 30}
    o = oracle_epoch(s, "srtf", reassign=prm)
    for g in run(s, prm):
        same(o, g)


def test_reassign_off_reports_nothing():
    nalar = _nalar()
    s = c4()
    ctx = nalar.Context.for_snapshot(s)
    ctx.upload(s)
    ctx.epoch("srtf")
    assert ctx.fetch()["n_reassign"] == 0
    ctx.set_policy_params(reassign=True, u_hi_pct=80, u_lo_pct=30)
    ctx.epoch("srtf")
    assert ctx.fetch()["n_reassign"] >= 1
    ctx.set_policy_params(reassign=False)
    ctx.epoch("srtf")
    assert ctx.fetch()["n_reassign"] == 0
    with pytest.raises(nalar.NalarError):
        ctx.set_policy_params(reassign=True, u_hi_pct=20, u_lo_pct=30)
    ctx.close()


@pytest.mark.parametrize("G", [2, 4])
def test_reassign_sharded_identical_on_every_rank(G):
    """G-invariance (I8): every rank reports the oracle's global commands."""
    import torch
    from tests.test_parity_gpu import _CAI
    from paper_2601_05109_b200.sharding import shard_bounds
    nalar = _nalar()
    s = c4(2)
    prm = {"u_hi_pct": 80, "u_lo_pct": 30}
    o = oracle_epoch(s, "srtf", reassign=prm)
    ctxs = []
    for k, (w0, w1) in enumerate(shard_bounds(s.wf_fut_off, G)):
        ctx = nalar.Context.for_snapshot(s, world=G, rank=k, collective=nalar.NALAR_COLL_EXTERNAL)
        ctx.set_policy_params(reassign=True, u_hi_pct=80, u_lo_pct=30)
        ctx.upload(s.slice_workflows(w0, w1))
        ctx.begin("srtf")
        ctxs.append(ctx)
    torch.cuda.synchronize()
    bufs = [torch.as_tensor(_CAI(*c.exchange_buffer()), device="cuda") for c in ctxs]
    total = torch.stack([b.to(torch.int64) for b in bufs]).sum(0).to(torch.int32)
    for b in bufs:
        b.copy_(total)
    torch.cuda.synchronize()
    for ctx in ctxs:
        ctx.finish()
        g = ctx.fetch()
        assert np.array_equal(g["ra_kill"], o["ra_kill"]) and np.array_equal(g["ra_prov"], o["ra_prov"])
        assert np.array_equal(g["t_busy"], o["t_busy"]) and np.array_equal(g["t_capsum"], o["t_cap"])
        ctx.close()


def test_next_rows_accepted_multi_rank():
    """NEXT-1 / NEXT-2 / NEXT-4 all run across ranks (tests/test_migrate_gpu.py,
    tests/test_batch_gpu.py, above)."""
    nalar = _nalar()
    s = c2(1)
    ctx = nalar.Context.for_snapshot(s, world=2, rank=0, collective=nalar.NALAR_COLL_EXTERNAL)
    ctx.set_policy_params(migrate=True)
    ctx.set_policy_params(t_max_batch=[4, 0, 0, 0], n_types=4)
    ctx.set_policy_params(reassign=True)
    ctx.close()
