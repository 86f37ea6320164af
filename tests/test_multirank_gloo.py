"""World-size-2/3 CPU tests (gloo) of the multi-GPU host logic.

The kernels need a GPU; what is tested here on CPU with real multi-process
collectives is everything around them: shard bounds, shard slicing, the NCCL
unique-id broadcast, the exchange-buffer layout (rank s fills only slot s of
H[G][R][Lv], plus per-instance in-flight loads), the allreduce, and the
global-rank formula DESIGN.md §5 derives from the reduced buffer --
evaluated here by a small host model and checked against the full-table oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from nalar_gen import c2, random_table, swe_table

S_DEF, S_ASG = 6, 7


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _table(which):
    return {"c2": lambda: c2(3, n_workflows=300),
            "swe": lambda: swe_table(12000, seed=4),
            "rand": lambda: random_table(5, n_workflows=30, max_rows=20, n_types=3,
                                         inst_per_type=(1, 3), max_cap=4)}[which]()


def _slots(spare2):
    s = [(sv, i) for i, sp in enumerate(spare2) for sv in range(1, sp + 1)]
    s.sort(key=lambda x: (-x[0], x[1]))
    return [i for _, i in s]


def _worker(rank, world, port, which, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle_epoch
        from paper_2601_05109_b200.sharding import exchange_words, shard_bounds, slot_view
        s = _table(which)
        o = oracle_epoch(s, "srtf")
        bounds = shard_bounds(s.wf_fut_off, world)
        w0, w1 = bounds[rank]
        sh = s.slice_workflows(w0, w1)
        r0 = sh.global_row_base
        I, T, Lv = s.n_instances, s.n_types, 256
        R = I + T
        # the NCCL id travels from rank 0 to every rank
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))
        # local contribution: slot `rank` of H + in-flight loads of local rows
        buf = np.zeros(exchange_words(world, R, Lv, I), np.int64)
        H, load, tot = slot_view(buf, world, R, Lv, I)
        local = []
        for lf in range(sh.n_futures):
            f = r0 + lf
            if sh.f_state[lf] in (1, 2):
                load[sh.f_executor[lf]] += 1
            if o["status"][f] in (S_DEF, S_ASG):
                r = int(sh.f_pin[lf]) if sh.f_pin[lf] >= 0 else I + int(sh.f_type[lf])
                H[rank, r, o["level"][f]] += 1
                tot[r] += 1
                local.append((lf, r, int(o["level"][f])))
        t = torch.from_numpy(buf)
        dist.all_reduce(t)
        buf = t.numpy()
        H, load, tot = slot_view(buf, world, R, Lv, I)
        assert np.array_equal(tot, H.sum(axis=(0, 2)))
        # every rank derives identical spare / bounds from the reduced buffer
        ld = s.i_base_load.astype(np.int64) + load
        spare = np.maximum(0, s.i_cap.astype(np.int64) - ld)
        assert np.array_equal(np.minimum(ld, 2**32 - 1), o["i_load"])
        admA = np.minimum(H[:, :I, :].sum(axis=(0, 2)), spare)
        spare2 = spare - admA
        Hg = H.sum(axis=0)
        above = np.concatenate([np.cumsum(Hg[:, ::-1], axis=1)[:, ::-1][:, 1:], np.zeros((R, 1), np.int64)],
                               axis=1)
        before = H[:rank].sum(axis=0)
        seen = {}
        got_asg = {}
        for lf, r, lv in local:            # rows in order => stable rank within (r, lv)
            k = seen.get((r, lv), 0)
            seen[(r, lv)] = k + 1
            g = above[r, lv] + before[r, lv] + k
            if r < I:
                if g < spare[r]:
                    got_asg[lf] = r
            else:
                inst = [i for i in range(I) if s.i_type[i] == r - I]
                sl = _slots([int(spare2[i]) for i in inst])
                if g < len(sl):
                    got_asg[lf] = inst[sl[g]]
        exp = {lf: int(o["instance"][r0 + lf]) for lf in range(sh.n_futures)
               if o["status"][r0 + lf] == S_ASG}
        assert got_asg == exp, (rank, len(got_asg), len(exp))
        q.put((rank, "ok", len(exp)))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("which", ["c2", "swe", "rand"])
def test_sharded_exchange_gloo(world, which):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, which, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    bad = [r for r in res if r[1] != "ok"]
    assert not bad, bad
    assert sum(r[2] for r in res) > 0 or which == "rand"


def test_shard_bounds_balanced():
    from paper_2601_05109_b200.sharding import shard_bounds
    s = swe_table(50000, seed=2)
    for G in (1, 2, 4, 8):
        b = shard_bounds(s.wf_fut_off, G)
        assert b[0][0] == 0 and b[-1][1] == s.n_workflows
        assert all(b[k][1] == b[k + 1][0] for k in range(G - 1))
        sizes = [int(s.wf_fut_off[w1]) - int(s.wf_fut_off[w0]) for w0, w1 in b]
        assert sum(sizes) == s.n_futures
        assert max(sizes) - min(sizes) <= 2 * int(np.diff(s.wf_fut_off.astype(np.int64)).max())
        # slices are self-contained and concatenate back to the table
        parts = [s.slice_workflows(w0, w1) for w0, w1 in b]
        assert np.array_equal(np.concatenate([p.f_state for p in parts]), s.f_state)
        for p in parts:
            e = p.edges & 0x7FFFFFFF
            assert (e < max(p.n_futures, 1)).all()


class _FakePeerCtx:
    """Stands in for a NALAR_COLL_PEER context: a per-rank IPC handle, and a
    record of what peer_connect received."""

    def __init__(self, rank):
        self.rank = rank
        self.got = None

    def peer_buffer(self):
        return 0x1000 * (self.rank + 1), bytes([self.rank]) * 64

    def peer_connect(self, ptrs=None, handles=None):
        self.got = (ptrs, handles)


def _peer_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_05109_b200.sharding import connect_peers
        ctx = _FakePeerCtx(rank)
        connect_peers(ctx)
        ptrs, handles = ctx.got
        assert ptrs is None
        assert handles == [bytes([r]) * 64 for r in range(world)], handles
        q.put((rank, "ok", 0))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_connect_peers_gathers_handles_in_rank_order(world):
    """sharding.connect_peers (NALAR_COLL_PEER across processes): every rank
    ends up with every rank's IPC handle, indexed by rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    bad = [r for r in res if r[1] != "ok"]
    assert not bad, bad


def test_connect_local_exchanges_pointers():
    from paper_2601_05109_b200.sharding import connect_local
    ctxs = [_FakePeerCtx(r) for r in range(4)]
    connect_local(ctxs)
    for c in ctxs:
        assert c.got[0] == [0x1000 * (r + 1) for r in range(4)] and c.got[1] is None
