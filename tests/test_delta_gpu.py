"""Delta mode on the GPU (nalar_delta_apply): the C3 dynamic router workload,
epoch after epoch, bit-exact against the oracle recomputing from scratch."""
import numpy as np
import pytest

from nalar_gen import RouterSim, c2, random_table
from oracle import oracle_epoch
from tests.test_delta_cpu import apply_delta_ref
from tests.test_parity_gpu import KEYS, assert_same

pytestmark = pytest.mark.gpu


def _ctx(n=120000, e=240000, w=12000, i=64, t=8, flags=0):
    from paper_2601_05109_b200 import nalar
    return nalar.Context(n, e, w, i, t, flags=flags)


@pytest.mark.parametrize("seed", [1, 2])
def test_router_trace_per_epoch_parity(seed):
    sim = RouterSim(seed)
    sim.warmup(450)
    s = sim.snapshot()
    ctx = _ctx()
    ctx.upload(s)
    for k in range(25):
        o = oracle_epoch(s, "srtf")
        ctx.epoch("srtf")
        g = ctx.fetch()
        assert_same(s, o, g, f"epoch {k}")
        d = sim.step(o["assign_row"], o["assign_inst"], o["new_pin"])
        ctx.apply_delta(d)
        s = sim.snapshot()
    ctx.close()


def _manual_delta(s, rng, o):
    """Updates, retirements, appends to live and new workflows, priority and
    instance updates on an arbitrary table (the simulator never sends the last two)."""
    from nalar_gen.dynamic import Delta
    W = s.n_workflows
    sizes = np.diff(s.wf_fut_off.astype(np.int64))
    live = [w for w in range(W)]
    ret = sorted(rng.choice(W, size=min(5, W), replace=False).tolist())
    d = Delta(flags=1)
    ups = []
    for w in rng.choice(W, size=min(20, W), replace=False).tolist():
        if sizes[w] and w not in ret:
            seq = int(rng.integers(0, sizes[w]))
            ups.append((int(s.wf_id[w]), seq, 3, -2, -2))          # resolve it
    if ups:
        d.upd_wf_id = np.array([u[0] for u in ups], np.uint64)
        d.upd_seq = np.array([u[1] for u in ups], np.uint32)
        d.upd_state = np.array([u[2] for u in ups], np.uint8)
        d.upd_executor = np.array([u[3] for u in ups], np.int16)
        d.upd_pin = np.array([u[4] for u in ups], np.int16)
    d.retired_wf_id = np.array([s.wf_id[w] for w in ret], np.uint64)
    aw, ap, ast, aty, ard, aex, apn, aeo, aed = [], [], [], [], [], [], [], [0], []
    keep = [w for w in live if w not in ret]
    grow = sorted(rng.choice(keep, size=min(6, len(keep)), replace=False).tolist())
    new_ids = [int(s.wf_id[-1]) + 5, int(s.wf_id[-1]) + 9]
    for wid, n0 in [(int(s.wf_id[w]), int(sizes[w])) for w in grow] + [(x, 0) for x in new_ids]:
        for j in range(int(rng.integers(1, 4))):
            seq = n0 + j
            aw.append(wid); ap.append(int(rng.integers(-2, 5))); ast.append(0)
            aty.append(int(rng.integers(0, s.n_types))); ard.append(int(rng.integers(0, 3)))
            aex.append(-1); apn.append(-1)
            if seq:
                aed.append(int(rng.integers(0, seq)))
                if rng.random() < 0.5:
                    aed.append(int(rng.integers(0, seq)) | (1 << 31))
            aeo.append(len(aed))
    d.app_wf_id = np.array(aw, np.uint64); d.app_wf_prio = np.array(ap, np.int32)
    d.app_state = np.array(ast, np.uint8); d.app_type = np.array(aty, np.uint8)
    d.app_round = np.array(ard, np.uint8); d.app_executor = np.array(aex, np.int16)
    d.app_pin = np.array(apn, np.int16); d.app_edge_off = np.array(aeo, np.uint32)
    d.app_edges = np.array(aed, np.uint32)
    d.prio_wf_id = np.array([s.wf_id[keep[0]], new_ids[0]], np.uint64)
    d.prio_value = np.array([7, -3], np.int32)
    d.inst_id = np.array([0, s.n_instances - 1], np.uint32)
    d.inst_cap = np.array([50, 0], np.uint32)
    d.inst_base_load = np.array([1, 3], np.uint32)
    return d


@pytest.mark.parametrize("seed", range(6))
def test_manual_deltas(seed):
    rng = np.random.default_rng(seed)
    s = c2(seed + 1, n_workflows=200) if seed % 2 == 0 else random_table(
        seed, n_workflows=60, max_rows=15, n_types=3, inst_per_type=(1, 4), max_cap=5)
    ctx = _ctx(w=2000, i=64, t=8)
    ctx.upload(s)
    for k in range(4):
        o = oracle_epoch(s, "lpt")
        ctx.epoch("lpt")
        assert_same(s, o, ctx.fetch(), f"epoch {k}")
        d = _manual_delta(s, rng, o)
        s2 = apply_delta_ref(s, o["assign_row"], o["assign_inst"], d)
        d.n_futures_after, d.n_workflows_after = s2.n_futures, s2.n_workflows
        ctx.apply_delta(d)
        s = s2
    o = oracle_epoch(s, "lpt")
    ctx.epoch("lpt")
    assert_same(s, o, ctx.fetch(), "final")


def test_delta_errors():
    from nalar_gen.dynamic import Delta
    from paper_2601_05109_b200 import nalar
    s = c2(1, n_workflows=50)
    ctx = _ctx(w=2000)
    ctx.upload(s)
    with pytest.raises(nalar.NalarError) as ei:              # APPLY_ASSIGNED before an epoch
        ctx.apply_delta(Delta(flags=1))
    assert ei.value.code == nalar.NALAR_E_STATE
    ctx.epoch("srtf")
    bad = Delta(flags=0, retired_wf_id=np.array([10**9], np.uint64))
    with pytest.raises(nalar.NalarError) as ei:
        ctx.apply_delta(bad)
    assert ei.value.code == nalar.NALAR_E_INVAL and ei.value.err_index == 0
    ctx.upload(s)
    bad = Delta(flags=0, upd_wf_id=np.array([s.wf_id[3], 10**9], np.uint64),
                upd_seq=np.array([0, 0], np.uint32), upd_state=np.array([3, 3], np.uint8),
                upd_executor=np.array([-2, -2], np.int16), upd_pin=np.array([-2, -2], np.int16))
    with pytest.raises(nalar.NalarError) as ei:
        ctx.apply_delta(bad)
    assert ei.value.code == nalar.NALAR_E_INVAL and ei.value.err_index == 1
    ctx.upload(s)
    # an appended edge that names a later future of its workflow -> K0 rejects the row
    bad = Delta(flags=0, app_wf_id=np.array([s.wf_id[0]], np.uint64),
                app_wf_prio=np.array([0], np.int32), app_state=np.array([0], np.uint8),
                app_type=np.array([0], np.uint8), app_round=np.array([0], np.uint8),
                app_executor=np.array([-1], np.int16), app_pin=np.array([-1], np.int16),
                app_edge_off=np.array([0, 1], np.uint32), app_edges=np.array([99], np.uint32))
    with pytest.raises(nalar.NalarError) as ei:
        ctx.apply_delta(bad)
    assert ei.value.code == nalar.NALAR_E_INVAL and ei.value.err_index == 10
    with pytest.raises(nalar.NalarError) as ei:               # table is now invalid
        ctx.epoch("srtf")
    assert ei.value.code == nalar.NALAR_E_STATE
