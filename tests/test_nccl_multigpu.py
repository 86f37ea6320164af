"""The library's NCCL world > 1 path on real GPUs: one process per GPU, the
communicator created by nalar_create from a broadcast nalar_nccl_unique_id,
the exchange buffer allreduced inside the epoch's CUDA graph, every rank's
decisions compared with the full-table oracle (global rank across shards,
DESIGN.md §5).  Also the peer-memory exchange across processes (CUDA IPC).

Needs at least two GPUs; skipped otherwise (the round's GPU box has one --
the same host logic runs world 2 / 3 on CPU in test_multirank_gloo.py, and the
kernels run with G ranks on one GPU in test_peer_gpu.py / test_parity_gpu.py).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _n_gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, which, collective, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from nalar_gen import c2, c4
        from oracle import oracle_epoch
        from paper_2601_05109_b200 import nalar
        from paper_2601_05109_b200.sharding import connect_peers, shard_bounds
        s = {"c2": lambda: c2(3), "c4": lambda: c4(2)}[which]()
        w0, w1 = shard_bounds(s.wf_fut_off, world)[rank]
        sh = s.slice_workflows(w0, w1)
        if collective == "nccl":
            obj = [nalar.nalar_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ctx = nalar.Context.for_snapshot(s, device=rank, world=world, rank=rank,
                                             collective=nalar.NALAR_COLL_NCCL, nccl_id=obj[0])
        else:
            ctx = nalar.Context.for_snapshot(s, device=rank, world=world, rank=rank,
                                             collective=nalar.NALAR_COLL_PEER)
            connect_peers(ctx)
        ctx.upload(sh)
        for _ in range(3):                    # direct launch, graph capture, graph replay
            ctx.epoch("srtf")
        g = ctx.fetch()
        ctx.close()
        o = oracle_epoch(s, "srtf")
        r0, r1 = sh.global_row_base, sh.global_row_base + sh.n_futures
        ok = all(np.array_equal(g[k], np.asarray(o[k])[r0:r1]) for k in ("status", "level", "depth", "instance"))
        ok &= all(np.array_equal(g[k], o[k]) for k in ("i_load", "i_spare", "i_assigned"))
        m = (o["assign_row"] >= r0) & (o["assign_row"] < r1)
        ok &= np.array_equal(g["assign_row"].astype(np.int64), o["assign_row"][m].astype(np.int64) - r0)
        q.put((rank, bool(ok), ""))
    except Exception as e:                    # reported to the parent
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs (NCCL world > 1 across processes)")
@pytest.mark.parametrize("collective", ["nccl", "peer"])
@pytest.mark.parametrize("which", ["c2", "c4"])
def test_world2_processes(collective, which):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, which, collective, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, ok, err in res:
        assert ok, (rank, err)
