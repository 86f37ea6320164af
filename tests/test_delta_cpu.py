"""The delta contract of include/nalar.h (nalar_delta_apply) on CPU.

A plain reference applier (written from the header's five steps) turns epoch
k's table + the oracle's decisions + the simulator's delta into a table that
must equal the simulator's own table of epoch k+1, row for row.  This pins the
delta format the GPU path consumes (tests/test_delta_gpu.py).
"""
import numpy as np
import pytest

from nalar_gen import CALL_BIT, QUEUED, RouterSim, Snapshot
from oracle import oracle_epoch


def apply_delta_ref(s: Snapshot, asg_rows, asg_inst, d) -> Snapshot:
    """The five steps of nalar_delta, on host arrays (test infrastructure)."""
    wids = [int(x) for x in s.wf_id]
    wf = {}
    for w, wid in enumerate(wids):
        a, b = int(s.wf_fut_off[w]), int(s.wf_fut_off[w + 1])
        rows = []
        for f in range(a, b):
            preds = [((int(v) & 0x7FFFFFFF) - a, bool(int(v) >> 31))
                     for v in s.edges[int(s.f_edge_off[f]):int(s.f_edge_off[f + 1])]]
            rows.append([int(s.f_state[f]), int(s.f_type[f]), int(s.f_round[f]),
                         int(s.f_executor[f]), int(s.f_pin[f]), preds])
        wf[wid] = [int(s.wf_prio[w]), rows]
    key = []
    for w, wid in enumerate(wids):
        key += [(wid, j) for j in range(int(s.wf_fut_off[w + 1] - s.wf_fut_off[w]))]
    if d.flags & 1:                                            # 1. assigned -> QUEUED
        for row, inst in zip(asg_rows, asg_inst):
            wid, j = key[int(row)]
            wf[wid][1][j][0], wf[wid][1][j][3] = QUEUED, int(inst)
    for k in range(len(d.upd_seq)):                            # 2. updates
        r = wf[int(d.upd_wf_id[k])][1][int(d.upd_seq[k])]
        if d.upd_state[k] != 0xFF:
            r[0] = int(d.upd_state[k])
        if d.upd_executor[k] != -2:
            r[3] = int(d.upd_executor[k])
        if d.upd_pin[k] != -2:
            r[4] = int(d.upd_pin[k])
    for wid in d.retired_wf_id:                                # 3. retire
        del wf[int(wid)]
    for k in range(len(d.app_wf_id)):                          # 4. append
        wid = int(d.app_wf_id[k])
        if wid not in wf:
            wf[wid] = [int(d.app_wf_prio[k]), []]
        preds = [(int(v) & 0x7FFFFFFF, bool(int(v) >> 31))
                 for v in d.app_edges[int(d.app_edge_off[k]):int(d.app_edge_off[k + 1])]]
        wf[wid][1].append([int(d.app_state[k]), int(d.app_type[k]), int(d.app_round[k]),
                           int(d.app_executor[k]), int(d.app_pin[k]), preds])
    for k in range(len(d.prio_wf_id)):                         # 5. priorities, instances
        wf[int(d.prio_wf_id[k])][0] = int(d.prio_value[k])
    cap, base = s.i_cap.copy(), s.i_base_load.copy()
    for k in range(len(d.inst_id)):
        cap[d.inst_id[k]], base[d.inst_id[k]] = d.inst_cap[k], d.inst_base_load[k]
    st, ty, rd, ex, pn, eoff, edges, off, prio, ids = [], [], [], [], [], [0], [], [0], [], []
    for wid in sorted(wf):
        p, rows = wf[wid]
        b0 = len(st)
        for r in rows:
            st.append(r[0]); ty.append(r[1]); rd.append(r[2]); ex.append(r[3]); pn.append(r[4])
            edges += [(b0 + q) | (int(CALL_BIT) if c else 0) for (q, c) in r[5]]
            eoff.append(len(edges))
        off.append(len(st)); prio.append(p); ids.append(wid)
    return Snapshot(wf_id=np.array(ids, np.uint64), wf_fut_off=np.array(off, np.uint32),
                    wf_prio=np.array(prio, np.int32), f_state=np.array(st, np.uint8),
                    f_type=np.array(ty, np.uint8), f_round=np.array(rd, np.uint8),
                    f_executor=np.array(ex, np.int16), f_pin=np.array(pn, np.int16),
                    f_edge_off=np.array(eoff, np.uint32), edges=np.array(edges, np.uint32),
                    i_type=s.i_type, i_cap=cap, i_base_load=base, t_affinity=s.t_affinity)


def same_table(a: Snapshot, b: Snapshot):
    for k, x in a.arrays().items():
        y = b.arrays()[k]
        assert x.shape == y.shape and np.array_equal(x, y), k


@pytest.mark.parametrize("seed", [1, 2])
def test_router_deltas_rebuild_the_next_table(seed):
    sim = RouterSim(seed, rps=40.0)
    sim.warmup(150)
    s = sim.snapshot()
    n_app = n_ret = n_upd = 0
    for _ in range(12):
        o = oracle_epoch(s, "srtf")
        d = sim.step(o["assign_row"], o["assign_inst"], o["new_pin"])
        nxt = sim.snapshot()
        same_table(apply_delta_ref(s, o["assign_row"], o["assign_inst"], d), nxt)
        assert d.n_futures_after == nxt.n_futures and d.n_workflows_after == nxt.n_workflows
        n_app += len(d.app_wf_id); n_ret += len(d.retired_wf_id); n_upd += len(d.upd_seq)
        s = nxt
    assert n_app > 0 and n_ret > 0 and n_upd > 0     # the trace is really dynamic
