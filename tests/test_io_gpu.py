"""The public API's kernel I/O paths (k_io.cu) against the oracle.

nalar_snapshot_upload moves pinned (device-mapped) host arrays with one
segment-copy kernel and falls back to cudaMemcpyAsync for pageable ones;
nalar_fetch_decisions writes pinned output buffers (and compacts the
assignment list) in one kernel.  Every combination must give bit-identical
results to the CPU oracle, and the size errors must still be reported.
"""
import numpy as np
import pytest

from nalar_gen import Snapshot, c1, c2, c4, random_table, swe_table
from oracle import oracle_epoch

pytestmark = pytest.mark.gpu

KEYS = ("status", "level", "depth", "instance", "new_pin", "wf_agg", "i_load", "i_spare",
        "i_assigned", "assign_row", "assign_inst", "kv_hint", "kv_level", "kv_home")


def _torch():
    import torch
    return torch


def pinned_like(a, keep):
    torch = _torch()
    t = torch.empty(max(a.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    keep.append(t)
    v = t.numpy()[:a.nbytes].view(a.dtype).reshape(a.shape)
    v[...] = a
    return v


def pinned_snapshot(s, keep, only=None):
    arrs = {k: (pinned_like(a, keep) if only is None or k in only else a) for k, a in s.arrays().items()}
    return Snapshot(global_row_base=s.global_row_base, name=s.name, **arrs)


def same(o, g, tag):
    for k in KEYS:
        a, b = np.asarray(o[k]), np.asarray(g[k])
        assert a.shape == b.shape and np.array_equal(a, b), f"{tag}: {k}"


@pytest.mark.parametrize("mk", [c1, lambda: c2(1), lambda: swe_table(3000, seed=5),
                                lambda: random_table(7, n_workflows=5, max_rows=30, consistent=True)])
@pytest.mark.parametrize("pin_in,pin_out", [(True, True), (True, False), (False, True)])
def test_pinned_paths_bit_exact(mk, pin_in, pin_out):
    from paper_2601_05109_b200 import nalar
    keep = []
    s = mk()
    o = oracle_epoch(s, "srtf")
    sp = pinned_snapshot(s, keep) if pin_in else s
    ctx = nalar.Context.for_snapshot(s)
    for _ in range(2):                       # re-upload into the same context
        ctx.upload(sp)
        ctx.epoch("srtf")
        alloc = (lambda n, dt: pinned_like(np.zeros(n, dt), keep)) if pin_out else None
        g = ctx.fetch(out=ctx.output_buffers(alloc=alloc))
        same(o, g, f"{s.name} in={pin_in} out={pin_out}")
    ctx.close()


def test_partially_pinned_snapshot():
    from paper_2601_05109_b200 import nalar
    keep = []
    s = swe_table(5000, seed=9)
    o = oracle_epoch(s, "lpt")
    sp = pinned_snapshot(s, keep, only={"f_state", "edges", "wf_prio", "i_cap"})
    ctx = nalar.Context.for_snapshot(s)
    ctx.upload(sp)
    ctx.epoch("lpt")
    g = ctx.fetch(out=ctx.output_buffers(alloc=lambda n, dt: pinned_like(np.zeros(n, dt), keep)))
    same(o, g, "partial")
    ctx.close()


def test_pinned_fetch_list_too_small():
    from paper_2601_05109_b200 import nalar
    keep = []
    s = c2(2)
    o = oracle_epoch(s, "srtf")
    n_asg = len(o["assign_row"])
    assert n_asg > 1
    ctx = nalar.Context.for_snapshot(s)
    ctx.upload(pinned_snapshot(s, keep))
    ctx.epoch("srtf")
    out = ctx.output_buffers(("status", "assign"), alloc=lambda n, dt: pinned_like(np.zeros(n, dt), keep))
    out["assign_row"] = out["assign_row"][:n_asg - 1]
    out["assign_inst"] = out["assign_inst"][:n_asg - 1]
    with pytest.raises(nalar.NalarError) as e:
        ctx.fetch(("status", "assign"), out=out)
    assert e.value.code == nalar.NALAR_E_SIZE
    # exactly enough room works, through the same fast path
    out["assign_row"] = pinned_like(np.zeros(n_asg, np.uint32), keep)
    out["assign_inst"] = pinned_like(np.zeros(n_asg, np.int16), keep)
    g = ctx.fetch(("status", "assign"), out=out)
    assert np.array_equal(g["assign_row"], o["assign_row"])
    assert np.array_equal(g["assign_inst"], o["assign_inst"])
    assert np.array_equal(g["status"], o["status"])
    ctx.close()


def test_pinned_invalid_upload_reports_row():
    from paper_2601_05109_b200 import nalar
    keep = []
    s = c1()
    arrs = s.arrays()
    edges = arrs["edges"].copy()
    # an edge of row 5 pointing forward (row 9): the first offending row is 5
    e0 = int(arrs["f_edge_off"][5])
    edges[e0] = 9
    bad = Snapshot(global_row_base=0, name="bad", **{**arrs, "edges": edges})
    ctx = nalar.Context.for_snapshot(bad)
    with pytest.raises(nalar.NalarError) as e:
        ctx.upload(pinned_snapshot(bad, keep))
    assert e.value.err_row == 5
    ctx.close()


def test_c4_pinned_e2e_matches_oracle():
    """The configuration bench.py's e2e leg times: pinned C4 in and out."""
    from paper_2601_05109_b200 import nalar
    keep = []
    s = c4()
    o = oracle_epoch(s, "srtf")
    sp = pinned_snapshot(s, keep)
    ctx = nalar.Context.for_snapshot(s)
    ctx.upload(sp)
    ctx.epoch("srtf")
    outb = ctx.output_buffers(("status", "instance", "assign"),
                              alloc=lambda n, dt: pinned_like(np.zeros(n, dt), keep))
    g = ctx.fetch(("status", "instance", "assign"), out=outb)
    for k in ("status", "instance", "assign_row", "assign_inst"):
        assert np.array_equal(np.asarray(o[k]), np.asarray(g[k])), k
    ctx.close()


def test_pinned_misaligned_arrays_bytewise_path():
    """Host arrays at odd offsets inside one pinned buffer: the copy kernel's
    bytewise path (neither side 16-byte aligned) must give the same bits."""
    from paper_2601_05109_b200 import nalar
    torch = _torch()
    s = swe_table(4000, seed=13)
    o = oracle_epoch(s, "srtf")
    arrs = s.arrays()
    total = sum(a.nbytes + 19 for a in arrs.values()) + 64
    t = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    buf = t.numpy()
    off, views = 3, {}
    for k, a in arrs.items():
        itemsize = a.dtype.itemsize
        off += (-off) % itemsize                    # element-aligned, not 16-byte aligned
        if off % 16 == 0:
            off += itemsize
        v = buf[off:off + a.nbytes].view(a.dtype).reshape(a.shape)
        v[...] = a
        views[k] = v
        off += a.nbytes + 5
    sp = Snapshot(global_row_base=0, name="misaligned", **views)
    ctx = nalar.Context.for_snapshot(s)
    ctx.upload(sp)
    ctx.epoch("srtf")
    same(o, ctx.fetch(), "misaligned")
    ctx.close()


def test_validation_window_with_many_empty_workflows():
    """K0 finds each row's workflow from a window of offsets per block; many
    empty workflows inside one block overflow the window and the rows beyond
    it take the global search: a cross-workflow edge there is still caught."""
    from paper_2601_05109_b200 import nalar
    n_empty = 700
    rows_a, rows_b = 10, 10
    W = 2 + n_empty
    off = np.concatenate([[0], np.full(1, rows_a), np.full(n_empty, rows_a), [rows_a + rows_b]]).astype(np.uint32)
    N = rows_a + rows_b
    eoff = np.zeros(N + 1, np.uint32)
    edges = []
    for f in range(N):
        w0 = 0 if f < rows_a else rows_a
        if f > w0:
            edges.append(f - 1)                 # chain inside the workflow
        eoff[f + 1] = len(edges)
    bad_row = rows_a + 5
    edges = np.array(edges, np.uint32)
    edges[int(eoff[bad_row])] = 3               # into the first workflow
    s = Snapshot(global_row_base=0, name="empties",
                 wf_id=np.arange(1, W + 1, dtype=np.uint64), wf_fut_off=off, wf_prio=np.zeros(W, np.int32),
                 f_state=np.zeros(N, np.uint8), f_type=np.zeros(N, np.uint8), f_round=np.zeros(N, np.uint8),
                 f_executor=np.full(N, -1, np.int16), f_pin=np.full(N, -1, np.int16), f_edge_off=eoff,
                 edges=edges, i_type=np.zeros(2, np.uint8), i_cap=np.full(2, 4, np.uint32),
                 i_base_load=np.zeros(2, np.uint32), t_affinity=np.zeros(1, np.uint8))
    ctx = nalar.Context.for_snapshot(s)
    with pytest.raises(nalar.NalarError) as e:
        ctx.upload(s)
    assert e.value.err_row == bad_row
    # the same table with the edge kept inside its workflow is accepted and exact
    good = s.arrays()
    good_edges = good["edges"].copy()
    good_edges[int(eoff[bad_row])] = bad_row - 1
    sg = Snapshot(global_row_base=0, name="empties-ok", **{**good, "edges": good_edges})
    ctx.upload(sg)
    ctx.epoch("srtf")
    same(oracle_epoch(sg, "srtf"), ctx.fetch(), "empties")
    ctx.close()
