"""The rank exchange over peer memory (NALAR_COLL_PEER, k_peer.cu) against the
full-table oracle.

G ranks are driven by one process on the one GPU: one context per rank, each
on its own stream, receive buffers exchanged as device pointers
(sharding.connect_local).  The epochs of all ranks are enqueued back to back
and run concurrently; each rank's gather kernel waits for every rank's flag.
The multi-process path differs only in how the buffers are opened (CUDA IPC
handles, sharding.connect_peers; its host logic is covered by the gloo test).
"""
import time

import numpy as np
import pytest

from nalar_gen import c2, c4, random_table, swe_table
from oracle import oracle_epoch

pytestmark = pytest.mark.gpu


def _ranks(s, G, flags=0):
    import torch
    from paper_2601_05109_b200 import nalar
    from paper_2601_05109_b200.sharding import connect_local, shard_bounds
    streams = [torch.cuda.Stream() for _ in range(G)]
    ctxs, shards = [], []
    for k, (w0, w1) in enumerate(shard_bounds(s.wf_fut_off, G)):
        ctxs.append(nalar.Context.for_snapshot(s, world=G, rank=k, collective=nalar.NALAR_COLL_PEER,
                                               stream=streams[k].cuda_stream, flags=flags))
        shards.append(s.slice_workflows(w0, w1))
    connect_local(ctxs)
    return ctxs, shards, streams


def _check(o, outs, tag):
    for k in ("status", "level", "depth", "instance", "new_pin", "wf_agg", "kv_hint", "kv_level", "kv_home"):
        got = np.concatenate([g[k] for g, _ in outs])
        assert np.array_equal(got, np.asarray(o[k])), (tag, k)
    for g, sh in outs:
        for k in ("i_load", "i_spare", "i_assigned"):
            assert np.array_equal(g[k], o[k]), (tag, k)
        r0, r1 = sh.global_row_base, sh.global_row_base + sh.n_futures
        m = (o["assign_row"] >= r0) & (o["assign_row"] < r1)
        assert np.array_equal(g["assign_row"].astype(np.int64), o["assign_row"][m].astype(np.int64) - r0), tag
        assert np.array_equal(g["assign_inst"], o["assign_inst"][m]), tag


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("which", ["c2", "c4", "rand"])
def test_peer_exchange_equals_single(G, which):
    s = {"c2": lambda: c2(2), "c4": lambda: c4(3),
         "rand": lambda: random_table(77, n_workflows=40, max_rows=25, n_types=3,
                                      inst_per_type=(1, 3), max_cap=4)}[which]()
    o = oracle_epoch(s, "srtf")
    ctxs, shards, _ = _ranks(s, G)
    for c, sh in zip(ctxs, shards):
        c.upload(sh)
    for _ in range(3):                      # direct launch, graph capture, graph replay
        for c in ctxs:
            c.epoch("srtf")
    _check(o, [(c.fetch(), sh) for c, sh in zip(ctxs, shards)], f"G={G} {which}")
    for c in ctxs:
        c.close()


def test_peer_exchange_policies_reupload_and_no_graph():
    """Epoch numbering and buffer parity across many epochs, policies, a
    re-upload of other tables, and direct launches."""
    from paper_2601_05109_b200 import nalar
    tables = [swe_table(6000, seed=11), swe_table(6000, seed=12)]
    for flags in (0, nalar.NALAR_F_NO_GRAPH):
        G = 3
        ctxs, _, _ = _ranks(tables[0], G, flags=flags)
        for rep in range(2):
            for s in tables:
                from paper_2601_05109_b200.sharding import shard_bounds
                shards = [s.slice_workflows(w0, w1) for w0, w1 in shard_bounds(s.wf_fut_off, G)]
                for c, sh in zip(ctxs, shards):
                    c.upload(sh)
                for pol in ("srtf", "lpt", "fcfs", "srtf"):
                    for c in ctxs:
                        c.epoch(pol)
                    _check(oracle_epoch(s, pol), [(c.fetch(), sh) for c, sh in zip(ctxs, shards)],
                           f"flags={flags} rep={rep} {pol}")
        for c in ctxs:
            c.close()


def test_peer_missing_rank_times_out_with_error():
    """A rank that never runs its epoch: the others' gather gives up after
    the timeout and their next fetch reports NALAR_E_COMM (no hang)."""
    from paper_2601_05109_b200 import nalar
    s = c2(1)
    ctxs, shards, _ = _ranks(s, 2, flags=nalar.NALAR_F_NO_GRAPH)
    for c, sh in zip(ctxs, shards):
        c.upload(sh)
    t0 = time.time()
    ctxs[0].epoch("srtf")
    with pytest.raises(nalar.NalarError) as e:
        ctxs[0].fetch()
    assert e.value.code == nalar.NALAR_E_COMM
    assert time.time() - t0 >= 4.0
    for c in ctxs:
        c.close()


def test_peer_requires_connect():
    from paper_2601_05109_b200 import nalar
    s = c2(1)
    ctx = nalar.Context.for_snapshot(s, world=2, rank=0, collective=nalar.NALAR_COLL_PEER)
    ctx.upload(s.slice_workflows(0, s.n_workflows // 2))
    with pytest.raises(nalar.NalarError) as e:
        ctx.epoch("srtf")
    assert e.value.code == nalar.NALAR_E_STATE
    ptr, handle = ctx.peer_buffer()
    assert ptr and len(handle) == 64
    ctx.close()


def _ipc_worker(rank, world, port, q):
    import os
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2601_05109_b200 import nalar
        from paper_2601_05109_b200.sharding import connect_peers, shard_bounds
        s = swe_table(8000, seed=21)
        o = oracle_epoch(s, "srtf")
        w0, w1 = shard_bounds(s.wf_fut_off, world)[rank]
        sh = s.slice_workflows(w0, w1)
        ctx = nalar.Context.for_snapshot(s, world=world, rank=rank, collective=nalar.NALAR_COLL_PEER)
        connect_peers(ctx)                      # CUDA IPC handles over gloo
        ctx.upload(sh)
        for _ in range(3):
            ctx.epoch("srtf")
        g = ctx.fetch()
        r0, r1 = sh.global_row_base, sh.global_row_base + sh.n_futures
        for k in ("status", "level", "instance"):
            assert np.array_equal(g[k], np.asarray(o[k])[r0:r1]), k
        for k in ("i_load", "i_spare", "i_assigned"):
            assert np.array_equal(g[k], o[k]), k
        m = (o["assign_row"] >= r0) & (o["assign_row"] < r1)
        assert np.array_equal(g["assign_row"].astype(np.int64), o["assign_row"][m].astype(np.int64) - r0)
        dist.barrier()
        ctx.close()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_across_processes_ipc():
    """Two processes (both on the one GPU), receive buffers opened by CUDA IPC
    handles exchanged with sharding.connect_peers -- the multi-process path
    bench.py takes for N > 1."""
    import socket
    import torch.multiprocessing as mp
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
    bad = [r for r in res if r[1] != "ok"]
    assert not bad, bad


@pytest.mark.parametrize("G", [2, 4])
def test_peer_exchange_with_reassignment(G):
    """NEXT-2 over the peer exchange: every rank reports the oracle's global
    kill / provision commands (the type statistics are built from the gathered
    buffer, identical on every rank)."""
    s = c4(2)
    o = oracle_epoch(s, "srtf", reassign={"u_hi_pct": 80, "u_lo_pct": 30})
    ctxs, shards, _ = _ranks(s, G)
    for c, sh in zip(ctxs, shards):
        c.set_policy_params(reassign=True, u_hi_pct=80, u_lo_pct=30)
        c.upload(sh)
    for _ in range(3):
        for c in ctxs:
            c.epoch("srtf")
    outs = [(c.fetch(), sh) for c, sh in zip(ctxs, shards)]
    _check(o, outs, f"reassign G={G}")
    for g, _ in outs:
        assert np.array_equal(g["ra_kill"], o["ra_kill"]) and np.array_equal(g["ra_prov"], o["ra_prov"])
        assert np.array_equal(g["t_busy"], o["t_busy"]) and np.array_equal(g["t_capsum"], o["t_cap"])
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("levels", [1, 7, 256])
def test_peer_exchange_levels(levels):
    """Other level counts change the slot size (R x Lv): layout offsets on
    both sides of the exchange must agree."""
    import torch
    from paper_2601_05109_b200 import nalar
    from paper_2601_05109_b200.sharding import connect_local, shard_bounds
    s = swe_table(7000, seed=31)
    o = oracle_epoch(s, "srtf", levels=levels)
    G = 3
    streams = [torch.cuda.Stream() for _ in range(G)]
    ctxs, shards = [], []
    for k, (w0, w1) in enumerate(shard_bounds(s.wf_fut_off, G)):
        ctxs.append(nalar.Context.for_snapshot(s, world=G, rank=k, collective=nalar.NALAR_COLL_PEER,
                                               stream=streams[k].cuda_stream, levels=levels))
        shards.append(s.slice_workflows(w0, w1))
    connect_local(ctxs)
    for c, sh in zip(ctxs, shards):
        c.upload(sh)
    for _ in range(2):
        for c in ctxs:
            c.epoch("srtf")
    _check(o, [(c.fetch(), sh) for c, sh in zip(ctxs, shards)], f"levels={levels}")
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("seed", range(12))
def test_peer_exchange_random_tables(seed):
    """Random small tables (pins, mixed affinities, empty shards at larger G)
    over the peer exchange, three policies."""
    G = 2 + seed % 6
    s = random_table(300 + seed, n_workflows=4 + seed % 9, max_rows=6 + seed % 20, n_types=1 + seed % 3,
                     inst_per_type=(1, 3), consistent=seed % 2 == 0, max_cap=2 + seed % 7, p_pin=0.3)
    pol = ["fcfs", "srtf", "lpt"][seed % 3]
    o = oracle_epoch(s, pol)
    ctxs, shards, _ = _ranks(s, G)
    for c, sh in zip(ctxs, shards):
        c.upload(sh)
    for _ in range(2):
        for c in ctxs:
            c.epoch(pol)
    _check(o, [(c.fetch(), sh) for c, sh in zip(ctxs, shards)], f"seed={seed} G={G}")
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("G", [2, 3])
def test_ranks_out_of_order_rejected(G):
    """Shards uploaded to the wrong ranks (the global rank is the row order
    across ranks, SURVEY 8(b) E_INVAL case): every rank's fetch reports
    NALAR_E_INVAL instead of silently mis-ranked admissions; in order again,
    the same contexts are bit-exact."""
    from paper_2601_05109_b200 import nalar
    s = swe_table(9000, seed=17)
    ctxs, shards, _ = _ranks(s, G)
    rev = shards[::-1]
    for c, sh in zip(ctxs, rev):
        c.upload(sh)
    for c in ctxs:
        c.epoch("srtf")
    for c in ctxs:
        with pytest.raises(nalar.NalarError) as e:
            c.fetch()
        assert e.value.code == nalar.NALAR_E_INVAL
    o = oracle_epoch(s, "srtf")
    for c, sh in zip(ctxs, shards):
        c.upload(sh)
    for c in ctxs:
        c.epoch("srtf")
    _check(o, [(c.fetch(), sh) for c, sh in zip(ctxs, shards)], "in order again")
    for c in ctxs:
        c.close()
