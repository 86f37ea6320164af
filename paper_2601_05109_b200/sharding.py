"""Host-side sharding of the future table by workflow id (multi-GPU).

Every dependency edge stays inside its workflow (Q1), so contiguous
workflow ranges are independent for the sweep; ranks exchange only the
(resource, level) histogram slots and per-instance in-flight counts.  Shards
are contiguous in row order, balanced by future count: shard k starts at the
first workflow w with wf_fut_off[w] >= k * N / G.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(wf_fut_off: np.ndarray, G: int) -> list[tuple[int, int]]:
    """Workflow ranges [(w0, w1), ...] of the G shards (some may be empty)."""
    off = np.asarray(wf_fut_off, dtype=np.int64)
    W = len(off) - 1
    N = int(off[-1]) if W >= 0 else 0
    starts = [0]
    for k in range(1, G):
        target = -(-k * N // G)                 # ceil(k * N / G)
        w = int(np.searchsorted(off[:W], target, side="left"))
        starts.append(max(w, starts[-1]))
    starts.append(W)
    return [(starts[k], starts[k + 1]) for k in range(G)]


def exchange_words(G: int, R: int, levels: int, n_inst: int) -> int:
    """u32 words of the per-epoch exchange buffer: H[G][R][Lv], load[I], tot[R],
    then (global_row_base, rows) per rank (the library checks that the ranks'
    shards are consecutive in the global row order)."""
    return G * R * levels + n_inst + R + 2 * G


def slot_view(buf: np.ndarray, G: int, R: int, levels: int, n_inst: int):
    """(H[G][R][Lv], load[I], tot[R]) views of an exchange buffer (host side)."""
    n = G * R * levels
    return buf[:n].reshape(G, R, levels), buf[n:n + n_inst], buf[n + n_inst:n + n_inst + R]


def connect_peers(ctx, group=None) -> None:
    """NALAR_COLL_PEER across processes: every rank publishes the CUDA IPC
    handle of its receive buffer, gathers everyone's (ordered by rank) and
    opens them in its context.  Collective over ``group`` (any backend that
    carries Python objects, e.g. gloo or nccl)."""
    import torch.distributed as dist
    _, handle = ctx.peer_buffer()
    world = dist.get_world_size(group)
    got = [None] * world
    dist.all_gather_object(got, (dist.get_rank(group), handle), group=group)
    handles = [None] * world
    for r, h in got:
        handles[r] = h
    ctx.peer_connect(handles=handles)


def connect_local(ctxs) -> None:
    """NALAR_COLL_PEER for ranks driven by one process (one context per rank,
    in rank order): the receive buffers are exchanged as device pointers."""
    ptrs = [c.peer_buffer()[0] for c in ctxs]
    for c in ctxs:
        c.peer_connect(ptrs=ptrs)
