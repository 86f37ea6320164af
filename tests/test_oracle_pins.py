"""Pins of the CPU oracle against what the paper and mathematics fix.

Each test pins the oracle to something other than itself: a hand-derived
golden file, brute-force enumeration, closed forms, SPEC worked examples and
invariants.  Citations: P:n = PAPER.md line n; S:n = SPEC.md line n.
"""
import os

import numpy as np
import pytest

from nalar_gen import (AFF_NONE, AFF_SESSION, AFF_STATEFUL, FAILED, PENDING, QUEUED, RESOLVED,
                       RUNNING, TableBuilder, c1, c2, c4, random_table)
from oracle import oracle_epoch, oracle_validate
from tests import bruteforce as bf

GOLD = os.path.join(os.path.dirname(__file__), "golden", "c1_srtf.txt")
S_RES, S_FAIL, S_INF, S_WAIT, S_DOOM, S_INEL, S_DEF, S_ASG = range(8)


def _read_golden():
    rows, kv = [], {}
    for line in open(GOLD):
        line = line.split("#")[0].strip()
        if not line:
            continue
        parts = line.split()
        if parts[0].isdigit():
            rows.append([int(x) for x in parts[2:]])
        else:
            kv[parts[0]] = [int(x) for x in parts[1:]]
    return np.array(rows), kv


# --------------------------------------------------------------------------
# C1: hand-derived golden output (tests/golden/c1_srtf.txt)
# --------------------------------------------------------------------------
def test_c1_golden_srtf():
    rows, kv = _read_golden()
    o = oracle_epoch(c1(), "srtf")
    assert o["status"].tolist() == rows[:, 0].tolist()
    assert o["depth"].tolist() == rows[:, 1].tolist()
    assert o["level"].tolist() == rows[:, 2].tolist()
    assert o["instance"].tolist() == rows[:, 3].tolist()
    assert o["new_pin"].tolist() == rows[:, 4].tolist()
    assert o["wf_agg"][0].tolist() == kv["wf_agg"]
    assert o["i_load"].tolist() == kv["i_load"]
    assert o["i_spare"].tolist() == kv["i_spare"]
    assert o["i_assigned"].tolist() == kv["i_assigned"]
    assert o["assign_row"].tolist() == kv["assign_row"]
    assert o["assign_inst"].tolist() == kv["assign_inst"]
    assert set(o["status"].tolist()) == set(range(8))       # every status occurs


@pytest.mark.parametrize("pol,key", [("lpt", "lpt_level"), ("fcfs", "fcfs_level")])
def test_c1_golden_other_policies(pol, key):
    rows, kv = _read_golden()
    o = oracle_epoch(c1(), pol)
    assert o["level"].tolist() == kv[key]
    assert o["status"].tolist() == rows[:, 0].tolist()
    assert o["instance"].tolist() == rows[:, 3].tolist()


# --------------------------------------------------------------------------
# O1: depth / doom / readiness against brute force
# --------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(300))
def test_depth_doom_ready_bruteforce(seed):
    s = random_table(seed, n_workflows=3, max_rows=9, max_preds=3)
    o = oracle_epoch(s, "srtf")
    doomed = bf.doomed_by_reachability(s)
    for f in range(s.n_futures):
        assert o["depth"][f] == bf.depth_by_path_enumeration(s, f), (seed, f)
        st = int(s.f_state[f])
        ready = st == PENDING and not doomed[f] and all(
            s.f_state[p] == RESOLVED for (p, _) in bf.preds(s, f, "dep"))
        if st == RESOLVED:
            assert o["status"][f] == S_RES
        elif st == FAILED:
            assert o["status"][f] == S_FAIL
        elif st in (QUEUED, RUNNING):
            assert o["status"][f] == S_INF and o["instance"][f] == s.f_executor[f]
        elif doomed[f]:
            assert o["status"][f] == S_DOOM, (seed, f)
        elif not ready:
            assert o["status"][f] == S_WAIT, (seed, f)
        else:
            assert o["status"][f] in (S_INEL, S_DEF, S_ASG), (seed, f)


def _chain(n, prio=0, call_every=0, rounds=None):
    tb = TableBuilder(i_type=[0], i_cap=[0], i_base_load=[0], t_affinity=[AFF_NONE])
    rows = []
    for j in range(n):
        preds = [] if j == 0 else [(j - 1, bool(call_every and j % call_every == 0))]
        rows.append((PENDING, 0, 0 if rounds is None else rounds[j], -1, -1, preds))
    tb.add_workflow(1, prio, rows)
    return tb.build()


def test_depth_chain_closed_form_and_saturation():
    # a chain of n has depth n-1 at its tail; levels saturate at Lv-1 (Q7)
    s = _chain(300, prio=-5, call_every=7)
    o = oracle_epoch(s, "srtf")
    assert o["depth"].tolist() == list(range(300))
    assert o["level"].tolist() == [min(255, max(0, d - 5)) for d in range(300)]
    o = oracle_epoch(s, "srtf", levels=16)
    assert o["level"].max() == 15


def test_c2_depth_closed_form():
    # Financial Analyst shape: plan 0 / specialists 1 / summarize 2 (fan-out/fan-in)
    s = c2(seed=2, n_workflows=50)
    o = oracle_epoch(s, "srtf")
    assert o["depth"].reshape(50, 10).tolist() == [[0] + [1] * 8 + [2]] * 50


def test_readiness_spec_examples():
    # {d1,d2}: d1 delivered -> still waiting; both -> queued(ready);
    # a duplicated dependency is idempotent.
    def table(st1, st2, dup):
        tb = TableBuilder(i_type=[0], i_cap=[5], i_base_load=[0], t_affinity=[AFF_NONE])
        p = [(0, False), (1, False)] + ([(0, False)] if dup else [])
        tb.add_workflow(1, 0, [(st1, 0, 0, 0 if st1 == RUNNING else -1, -1, []),
                               (st2, 0, 0, 0 if st2 == RUNNING else -1, -1, []),
                               (PENDING, 0, 0, -1, -1, p)])
        return tb.build()
    assert oracle_epoch(table(RESOLVED, RUNNING, False))["status"][2] == S_WAIT
    assert oracle_epoch(table(RESOLVED, RESOLVED, False))["status"][2] == S_ASG
    assert oracle_epoch(table(RESOLVED, RESOLVED, True))["status"][2] == S_ASG
    # CALL edges do not gate readiness (Q2) but count for depth (Q4)
    tb = TableBuilder(i_type=[0], i_cap=[5], i_base_load=[0], t_affinity=[AFF_NONE])
    tb.add_workflow(1, 0, [(RUNNING, 0, 0, 0, -1, []), (PENDING, 0, 0, -1, -1, [(0, True)])])
    o = oracle_epoch(tb.build())
    assert o["status"][1] == S_ASG and o["depth"][1] == 1


# --------------------------------------------------------------------------
# O4 order: SPEC worked examples
# --------------------------------------------------------------------------
def _one_slot_table(entries, aff=AFF_NONE, cap=1):
    """entries: list of (prio, depth_chain_len, round) -> one workflow each whose
    last row is a ready future of type 0; one instance with `cap` spare."""
    tb = TableBuilder(i_type=[0], i_cap=[cap], i_base_load=[0], t_affinity=[aff])
    for w, (prio, d, rd) in enumerate(entries):
        rows = [(RESOLVED, 0, rd, 0, -1, [] if j == 0 else [(j - 1, False)]) for j in range(d)]
        rows.append((PENDING, 0, rd, -1, -1, [(d - 1, False)] if d else []))
        tb.add_workflow(w + 1, prio, rows)
    return tb.build()


def _winner(s, pol):
    o = oracle_epoch(s, pol)
    return [int(r) for r in np.nonzero(o["status"] == S_ASG)[0]]


def test_spec_priority_and_fifo():
    # S:284 queue [p=0 t=1, p=5 t=2] -> picks p=5 (set_priority P:389)
    s = _one_slot_table([(0, 0, 0), (5, 0, 0)])
    assert _winner(s, "fcfs") == [1]
    # S:285 equal priorities -> earlier one wins (tie-break by future id, Q8)
    s = _one_slot_table([(3, 0, 0), (3, 0, 0)])
    assert _winner(s, "fcfs") == [0]


def test_spec_srtf_depth():
    # S:464 futures at depths 1 and 3 -> depth-3 future first
    s = _one_slot_table([(0, 1, 0), (0, 3, 0)])
    assert _winner(s, "srtf") == [2 + 3]      # rows: w0 = 0..1, w1 = 2..5
    assert _winner(s, "fcfs") == [1]


def test_spec_lpt_reentry():
    # S:475 session with 2 requeues vs fresh -> requeued first
    s = _one_slot_table([(0, 0, 0), (0, 0, 2)])
    assert _winner(s, "lpt") == [1]
    assert _winner(s, "fcfs") == [0]


# --------------------------------------------------------------------------
# O6/O7 admission + placement: brute force on tiny tables
# --------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(400))
def test_admission_bruteforce(seed):
    s = random_table(1000 + seed, n_workflows=3, max_rows=5, n_types=2, inst_per_type=(0, 2),
                     max_cap=3, max_base=2)
    o = oracle_epoch(s, ["fcfs", "srtf", "lpt"][seed % 3])
    I = s.n_instances
    elig = [f for f in range(s.n_futures) if o["status"][f] in (S_DEF, S_ASG)]
    if len(elig) > 10:
        pytest.skip("too many for brute force")
    key = lambda f: (-int(o["level"][f]), f)
    order = sorted(elig, key=key)                   # library sort (O4 order)
    # load / spare from the definition, counted independently
    load = [int(s.i_base_load[i]) + sum(1 for f in range(s.n_futures)
                                         if s.f_state[f] in (QUEUED, RUNNING)
                                         and s.f_executor[f] == i) for i in range(I)]
    spare = [max(0, int(s.i_cap[i]) - load[i]) for i in range(I)]
    assert o["i_load"].tolist() == load and o["i_spare"].tolist() == spare
    # phase A: lexicographically greatest admitted set under per-pin capacity
    pinned = [f for f in order if s.f_pin[f] >= 0]
    admA = bf.lexmax_admission(pinned, {f: int(s.f_pin[f]) for f in pinned},
                               {i: spare[i] for i in range(I)})
    for f in pinned:
        assert (o["status"][f] == S_ASG) == (f in admA), (seed, f)
        if f in admA:
            assert o["instance"][f] == s.f_pin[f]
    spare2 = list(spare)
    for f in admA:
        spare2[int(s.f_pin[f])] -= 1
    # phase B per type: lexmax under the type's total spare; placement = slot list
    for t in range(s.n_types):
        inst = [i for i in range(I) if s.i_type[i] == t]
        unp = [f for f in order if s.f_pin[f] < 0 and s.f_type[f] == t]
        admB = bf.lexmax_admission(unp, {f: t for f in unp}, {t: sum(spare2[i] for i in inst)})
        slots = bf.slot_list([spare2[i] for i in inst])
        k = 0
        for f in unp:
            assert (o["status"][f] == S_ASG) == (f in admB), (seed, f)
            if f in admB:
                assert o["instance"][f] == inst[slots[k]], (seed, f)
                assert o["new_pin"][f] == int(s.t_affinity[t] != AFF_NONE)
                k += 1


@pytest.mark.parametrize("seed", range(200))
def test_water_fill_equals_slot_enumeration(seed):
    rng = np.random.default_rng(seed)
    n_i = int(rng.integers(1, 6))
    caps = rng.integers(0, 6, n_i)
    n_f = int(rng.integers(0, 20))
    tb = TableBuilder(i_type=[0] * n_i, i_cap=caps, i_base_load=[0] * n_i, t_affinity=[AFF_NONE])
    tb.add_workflow(1, 0, [(PENDING, 0, 0, -1, -1, [])] * n_f)
    o = oracle_epoch(tb.build(), "fcfs")
    got = [int(o["instance"][f]) for f in range(n_f) if o["status"][f] == S_ASG]
    assert got == bf.slot_list([int(c) for c in caps])[:n_f]


def test_water_fill_hand_check():
    # spares (3,1,3) -> i0,i2,i0,i2,i0,i1,i2
    assert bf.slot_list([3, 1, 3]) == [0, 2, 0, 2, 0, 1, 2]
    tb = TableBuilder(i_type=[0] * 3, i_cap=[3, 1, 3], i_base_load=[0] * 3, t_affinity=[AFF_NONE])
    tb.add_workflow(1, 0, [(PENDING, 0, 0, -1, -1, [])] * 8)
    o = oracle_epoch(tb.build(), "fcfs")
    assert o["instance"].tolist() == [0, 2, 0, 2, 0, 1, 2, -1]
    assert o["status"][7] == S_DEF


def test_spec_load_balance_examples():
    # S:434 queues (0,0) -> equal share; S:435 queues (4,0), C=4 -> all to the
    # idle instance; S:436 single instance -> everything to it.
    def run(caps, bases, n):
        tb = TableBuilder(i_type=[0] * len(caps), i_cap=caps, i_base_load=bases,
                          t_affinity=[AFF_NONE])
        tb.add_workflow(1, 0, [(PENDING, 0, 0, -1, -1, [])] * n)
        return oracle_epoch(tb.build(), "fcfs")["instance"].tolist()
    assert run([4, 4], [0, 0], 4) == [0, 1, 0, 1]
    assert run([4, 4], [4, 0], 4) == [1, 1, 1, 1]
    assert run([4], [0], 3) == [0, 0, 0]


def test_spec_pin_precedence_and_stateful():
    # a pinned session goes to its pin even when a peer has more spare.
    tb = TableBuilder(i_type=[0, 0], i_cap=[1, 5], i_base_load=[0, 0], t_affinity=[AFF_SESSION])
    tb.add_workflow(1, 0, [(PENDING, 0, 0, -1, 0, [])])
    o = oracle_epoch(tb.build())
    assert o["status"][0] == S_ASG and o["instance"][0] == 0 and o["new_pin"][0] == 0
    # S:256 / P:267: stateful -- a second future of the same session is not
    # placed while the first is in flight; then it goes to the same instance.
    tb = TableBuilder(i_type=[0, 0], i_cap=[5, 5], i_base_load=[0, 0], t_affinity=[AFF_STATEFUL])
    tb.add_workflow(1, 0, [(RUNNING, 0, 0, 1, 1, []), (PENDING, 0, 0, -1, 1, [])])
    o = oracle_epoch(tb.build())
    assert o["status"][1] == S_INEL
    tb = TableBuilder(i_type=[0, 0], i_cap=[5, 5], i_base_load=[0, 0], t_affinity=[AFF_STATEFUL])
    tb.add_workflow(1, 0, [(RESOLVED, 0, 0, 1, 1, []), (PENDING, 0, 0, -1, 1, []),
                           (PENDING, 0, 0, -1, 1, [])])
    o = oracle_epoch(tb.build())
    assert o["status"].tolist() == [S_RES, S_ASG, S_INEL] and o["instance"][1] == 1
    # stateful in-order: the lowest pending future must go first even if a
    # later one is ready (fence S:222)
    tb = TableBuilder(i_type=[0], i_cap=[5], i_base_load=[0], t_affinity=[AFF_STATEFUL])
    tb.add_workflow(1, 0, [(RUNNING, 0, 0, 0, -1, []), (PENDING, 0, 0, -1, -1, [(0, False)]),
                           (PENDING, 0, 0, -1, -1, [])])
    tb.add_workflow(2, 0, [(PENDING, 0, 0, -1, -1, []), (PENDING, 0, 0, -1, -1, [(0, True)])])
    o = oracle_epoch(tb.build())
    assert o["status"].tolist() == [S_INF, S_WAIT, S_INEL, S_ASG, S_INEL]
    # a doomed future never runs, so it does not fence its session (Q3, Q12)
    tb = TableBuilder(i_type=[0], i_cap=[5], i_base_load=[0], t_affinity=[AFF_STATEFUL])
    tb.add_workflow(1, 0, [(FAILED, 0, 0, 0, -1, []), (PENDING, 0, 0, -1, -1, [(0, False)]),
                           (PENDING, 0, 0, -1, -1, [])])
    o = oracle_epoch(tb.build())
    assert o["status"].tolist() == [S_FAIL, S_DOOM, S_ASG]


# --------------------------------------------------------------------------
# invariants I1-I10 on generated workloads
# --------------------------------------------------------------------------
def _check_invariants(s, o):
    N, I = s.n_futures, s.n_instances
    st = o["status"]
    # I10 conservation
    assert np.bincount(st, minlength=8).sum() == N
    agg = o["wf_agg"]
    assert agg[:, 0].sum() == N
    assert (agg[:, 1] + agg[:, 3] + agg[:, 4] + agg[:, 5] == agg[:, 0]).all()
    sizes = np.diff(s.wf_fut_off.astype(np.int64))
    assert (agg[:, 0] == sizes).all()
    asg = np.nonzero(st == S_ASG)[0]
    for f in asg:
        # I1 readiness safety
        assert s.f_state[f] == PENDING
        for (p, _) in bf.preds(s, int(f), "dep"):
            assert s.f_state[p] == RESOLVED
        # I7 pinned futures only go to their pin; instance type matches
        if s.f_pin[f] >= 0:
            assert o["instance"][f] == s.f_pin[f]
        assert s.i_type[o["instance"][f]] == s.f_type[f]
    # I2 capacity
    cnt = np.bincount(o["instance"][asg].astype(np.int64), minlength=I) if I else np.zeros(0)
    assert (cnt == o["i_assigned"]).all()
    load = o["i_load"].astype(np.int64)
    assert (load + cnt <= np.maximum(s.i_cap.astype(np.int64), load)).all()
    # I4 no inversion inside a resource, I5 work conservation
    after = o["i_spare"].astype(np.int64) - cnt
    assert (after >= 0).all()
    lv = o["level"].astype(np.int64)
    for f in np.nonzero(st == S_DEF)[0]:
        if s.f_pin[f] >= 0:
            same = asg[s.f_pin[asg] == s.f_pin[f]]
            assert after[s.f_pin[f]] == 0
        else:
            same = asg[(s.f_pin[asg] < 0) & (s.f_type[asg] == s.f_type[f])]
            assert (after[s.i_type == s.f_type[f]] == 0).all()
        for g in same:
            assert (lv[g], -g) > (lv[f], -f)
    # I6 stateful: at most one placed per (w, stateful type), none if one is in flight
    wf = np.repeat(np.arange(s.n_workflows), np.diff(s.wf_fut_off.astype(np.int64)))
    for t in np.nonzero(s.t_affinity == AFF_STATEFUL)[0]:
        for w in range(s.n_workflows):
            m = (wf == w) & (s.f_type == t)
            if (m & (st == S_ASG)).sum():
                assert (m & (st == S_ASG)).sum() == 1 and (m & (st == S_INF)).sum() == 0


@pytest.mark.parametrize("seed", range(150))
def test_invariants_random(seed):
    s = random_table(5000 + seed, n_workflows=6, max_rows=12, n_types=3, consistent=seed % 2 == 0)
    o = oracle_epoch(s, ["fcfs", "srtf", "lpt"][seed % 3])
    _check_invariants(s, o)


def test_invariants_c2_c4():
    for s in (c2(seed=1), c4(seed=2)):
        for pol in ("srtf", "lpt"):
            o = oracle_epoch(s, pol)
            _check_invariants(s, o)
            # I9 run-to-run bit identity
            o2 = oracle_epoch(s, pol)
            for k in ("status", "level", "depth", "instance", "new_pin", "assign_row"):
                assert (o[k] == o2[k]).all()


# --------------------------------------------------------------------------
# O2 aggregates and O3 eligibility re-derived from brute force (not from the
# oracle's statuses): every wf_agg field by numpy bincount over the workflow of
# each row, eligibility by scanning (w, t) groups in row order.
# P:338 [§4.1] aggregating metadata; P:267-268 [§3.4] stateful; P:575 [§5]
# managed state (Q12, Q13).
# --------------------------------------------------------------------------
def _bf_ready_doomed(s):
    doomed = np.array(bf.doomed_by_reachability(s), dtype=bool)
    ready = np.zeros(s.n_futures, dtype=bool)
    for f in range(s.n_futures):
        ready[f] = (s.f_state[f] == PENDING and not doomed[f]
                    and all(s.f_state[p] == RESOLVED for (p, _) in bf.preds(s, f, "dep")))
    return ready, doomed


def _bf_wf_agg(s):
    N, W = s.n_futures, s.n_workflows
    wf = np.repeat(np.arange(W), np.diff(s.wf_fut_off.astype(np.int64)))
    ready, doomed = _bf_ready_doomed(s)
    st = s.f_state
    depth = np.array([bf.depth_by_path_enumeration(s, f) for f in range(N)], dtype=np.int64)

    def count(mask):
        return np.bincount(wf[mask], minlength=W)

    def gmax(v):
        out = np.zeros(W, dtype=np.int64)
        np.maximum.at(out, wf, v) if N else None
        return out
    inflight = (st == QUEUED) | (st == RUNNING)
    return np.stack([count(np.ones(N, dtype=bool)), count(st == PENDING), count(ready),
                     count(inflight), count(st == RESOLVED), count(st == FAILED), count(doomed),
                     count((st == PENDING) & (s.f_pin >= 0)), gmax(depth),
                     gmax(s.f_round.astype(np.int64))], axis=1), ready, doomed


def _bf_eligible(s, ready, doomed):
    """Eligibility of each ready future by scanning its (workflow, type) group in
    row order: STATEFUL = nothing of the group in flight and the lowest-row
    PENDING non-doomed future; SESSION without a pin = the lowest-row ready
    unpinned future; otherwise eligible."""
    elig = np.zeros(s.n_futures, dtype=bool)
    for w in range(s.n_workflows):
        rows = range(int(s.wf_fut_off[w]), int(s.wf_fut_off[w + 1]))
        for f in rows:
            if not ready[f]:
                continue
            t = s.f_type[f]
            grp = [g for g in rows if s.f_type[g] == t]
            aff = s.t_affinity[t]
            if aff == AFF_STATEFUL:
                busy = any(s.f_state[g] in (QUEUED, RUNNING) for g in grp)
                first = min(g for g in grp if s.f_state[g] == PENDING and not doomed[g])
                elig[f] = not busy and first == f
            elif aff == AFF_SESSION and s.f_pin[f] < 0:
                elig[f] = min(g for g in grp if ready[g] and s.f_pin[g] < 0) == f
            else:
                elig[f] = True
    return elig


@pytest.mark.parametrize("seed", range(150))
def test_wf_agg_and_eligibility_bruteforce(seed):
    s = random_table(7000 + seed, n_workflows=2 + seed % 5, max_rows=3 + seed % 9,
                     n_types=1 + seed % 3, consistent=seed % 2 == 0, p_pin=0.6)
    o = oracle_epoch(s, ["fcfs", "srtf", "lpt"][seed % 3])
    agg, ready, doomed = _bf_wf_agg(s)
    assert o["wf_agg"].astype(np.int64).tolist() == agg.tolist(), seed
    elig = _bf_eligible(s, ready, doomed)
    st = o["status"]
    assert ((st == S_DEF) | (st == S_ASG)).tolist() == elig.tolist(), seed
    assert (st == S_INEL).tolist() == (ready & ~elig).tolist(), seed


def test_wf_agg_pinned_pending_counts_pending_only():
    # pinned_pending counts PENDING futures carrying a pin, whatever else they
    # are (a doomed pinned PENDING counts); pinned RESOLVED / RUNNING do not.
    tb = TableBuilder(i_type=[0, 0], i_cap=[4, 4], i_base_load=[0, 0], t_affinity=[AFF_SESSION])
    tb.add_workflow(1, 0, [(RESOLVED, 0, 0, 0, 0, []), (RUNNING, 0, 0, 0, 0, []),
                           (FAILED, 0, 0, 1, 1, []), (PENDING, 0, 0, -1, 1, [(2, False)]),
                           (PENDING, 0, 0, -1, 0, []), (PENDING, 0, 0, -1, -1, [])])
    o = oracle_epoch(tb.build())
    # total pending ready inflight resolved failed doomed pinned_pending maxd maxr
    assert o["wf_agg"][0].tolist() == [6, 3, 2, 1, 1, 1, 1, 2, 1, 0]


def test_session_first_placement_q13():
    # Q13 / P:575: an unpinned SESSION future places only as the lowest-row READY
    # unpinned future of its (w, t).  The lowest PENDING one (r1) is still
    # waiting on r0, so the later ready r2 is the first placement.
    tb = TableBuilder(i_type=[0, 0], i_cap=[4, 4], i_base_load=[0, 0], t_affinity=[AFF_SESSION])
    tb.add_workflow(1, 0, [(RUNNING, 0, 0, 0, -1, []), (PENDING, 0, 0, -1, -1, [(0, False)]),
                           (PENDING, 0, 0, -1, -1, []), (PENDING, 0, 0, -1, -1, [])])
    o = oracle_epoch(tb.build())
    assert o["status"].tolist() == [S_INF, S_WAIT, S_ASG, S_INEL]
    assert o["new_pin"].tolist() == [0, 0, 1, 0]
    # the first ready future carries a pin: it goes to its pin (phase A) and
    # does not take the first-placement slot; the lowest ready UNPINNED one does.
    tb = TableBuilder(i_type=[0, 0], i_cap=[4, 4], i_base_load=[0, 0], t_affinity=[AFF_SESSION])
    tb.add_workflow(1, 0, [(PENDING, 0, 0, -1, 1, []), (PENDING, 0, 0, -1, -1, []),
                           (PENDING, 0, 0, -1, -1, [])])
    o = oracle_epoch(tb.build())
    assert o["status"].tolist() == [S_ASG, S_ASG, S_INEL]
    assert o["instance"][0] == 1 and o["new_pin"].tolist() == [0, 1, 0]
    # a doomed future is not ready, so it never takes the slot
    tb = TableBuilder(i_type=[0, 0], i_cap=[4, 4], i_base_load=[0, 0], t_affinity=[AFF_SESSION])
    tb.add_workflow(1, 0, [(FAILED, 0, 0, 0, -1, []), (PENDING, 0, 0, -1, -1, [(0, False)]),
                           (PENDING, 0, 0, -1, -1, [])])
    o = oracle_epoch(tb.build())
    assert o["status"].tolist() == [S_FAIL, S_DOOM, S_ASG]


# --------------------------------------------------------------------------
# input contract (Q1): invalid tables are rejected with the first bad row
# --------------------------------------------------------------------------
def test_validation():
    assert oracle_validate(c1()) == (0, -1)
    s = c1(); s.edges[3] = 23                      # row 3 (test0) -> later row
    assert oracle_validate(s) == (-1, 3)
    s = c1(); s.f_pin[7] = 0                       # TOOL future pinned to an LLM instance
    assert oracle_validate(s) == (-1, 7)
    s = c1(); s.f_executor[3] = -1                 # RUNNING without executor
    assert oracle_validate(s) == (-1, 3)
    s = c1(); s.f_state[4] = 9
    assert oracle_validate(s) == (-1, 4)
    s = c2(seed=1, n_workflows=3); s.edges[-1] = 5  # edge into another workflow
    assert oracle_validate(s)[0] == -1 and oracle_validate(s)[1] == 29
    s = c2(seed=1, n_workflows=3); s.wf_id[2] = s.wf_id[1]
    assert oracle_validate(s) == (-1, -1)


# --------------------------------------------------------------------------
# O9 K,V-cache retention hints (NEXT-3, SPEC kv_hint S:542)
# --------------------------------------------------------------------------
KV_NONE, KV_RETAIN, KV_OFFLOAD, KV_DROP = range(4)


def test_kv_hints_hand_derived():
    """Every hint class, derived by hand.  Types: 0 LLM (SESSION), 1 TOOL
    (NONE), 2 CODER (SESSION); instances 0,1 LLM; 2 TOOL; 3,4 CODER."""
    tb = TableBuilder(i_type=[0, 0, 1, 2, 2], i_cap=[4, 4, 4, 4, 4], i_base_load=[0] * 5,
                      t_affinity=[AFF_SESSION, AFF_NONE, AFF_SESSION])
    # w0: LLM session homed at min(1, 0) = 0 with a live PENDING future (level =
    # prio 5 + SRTF depth 1 = 6) -> retain@0, level 6.  CODER session homed at 4,
    # only RESOLVED -> offload (the workflow is still live).
    tb.add_workflow(1, 5, [(RESOLVED, 0, 0, -1, 1, []),            # r0 LLM pinned 1
                           (PENDING, 0, 0, -1, 0, [(0, False)]),    # r1 LLM pinned 0, ready, depth 1
                           (RESOLVED, 2, 0, -1, 4, [(0, False)]),   # r2 CODER pinned 4
                           (PENDING, 1, 0, -1, -1, [(2, False)])])  # r3 TOOL
    # w1: everything terminal -> its LLM session (home 1) is dropped; its CODER
    # session has no pin -> no hint.
    tb.add_workflow(2, 0, [(RESOLVED, 0, 0, -1, 1, []),
                           (FAILED, 2, 0, -1, -1, [(0, False)])])
    # w2: LLM session homed at 1 whose only PENDING future is doomed (a FAILED DEP
    # predecessor); the TOOL future is RUNNING -> offload.  CODER session pinned
    # at 3 with a QUEUED future at 3 (level = prio 0 + depth 0) -> retain@3.
    tb.add_workflow(3, 0, [(FAILED, 1, 0, -1, -1, []),
                           (PENDING, 0, 0, -1, 1, [(0, False)]),
                           (RUNNING, 1, 0, 2, -1, []),
                           (QUEUED, 2, 0, 3, 3, [])])
    s = tb.build()
    o = oracle_epoch(s, "srtf")
    assert o["kv_hint"].tolist() == [[KV_RETAIN, KV_NONE, KV_OFFLOAD],
                                     [KV_DROP, KV_NONE, KV_NONE],
                                     [KV_OFFLOAD, KV_NONE, KV_RETAIN]]
    assert o["kv_home"].tolist() == [[0, -1, 4], [1, -1, -1], [1, -1, 3]]
    assert o["kv_level"].tolist() == [[6, 0, 0], [0, 0, 0], [0, 0, 0]]
    assert o["status"][[1, 7]].tolist() == [S_ASG, S_DOOM]


def _kv_from_statuses(s, o):
    """O9 by another route: live futures are read off the O8 statuses (INFLIGHT,
    WAITING, INELIGIBLE, DEFERRED, ASSIGNED -- not DOOMED), homes by a vectorised
    grouped minimum, levels by a grouped maximum."""
    W, T = s.n_workflows, s.n_types
    wf = np.repeat(np.arange(W), np.diff(s.wf_fut_off.astype(np.int64)))
    ty = s.f_type.astype(np.int64)
    live = np.isin(o["status"], [S_INF, S_WAIT, S_INEL, S_DEF, S_ASG])
    key = wf * T + ty
    home = np.full(W * T, 1 << 30, np.int64)
    pinned = s.f_pin >= 0
    np.minimum.at(home, key[pinned], s.f_pin[pinned].astype(np.int64))
    n_live = np.bincount(key[live], minlength=W * T)
    lev = np.zeros(W * T, np.int64)
    np.maximum.at(lev, key[live], o["level"][live].astype(np.int64))
    wf_live = np.bincount(wf[live], minlength=W)[np.arange(W * T) // T]
    sess = (s.t_affinity[np.arange(W * T) % T] == AFF_SESSION)
    has_home = sess & (home < (1 << 30))
    hint = np.where(~has_home, KV_NONE,
                    np.where(n_live > 0, KV_RETAIN, np.where(wf_live > 0, KV_OFFLOAD, KV_DROP)))
    lev = np.where(sess, lev, 0)
    home = np.where(has_home, home, -1)
    return hint.reshape(W, T), lev.reshape(W, T), home.reshape(W, T)


@pytest.mark.parametrize("seed", range(150))
def test_kv_hints_grouped_route(seed):
    s = random_table(seed, n_workflows=1 + seed % 6, max_rows=2 + seed % 25, n_types=1 + seed % 4,
                     inst_per_type=(0, 1 + seed % 3), consistent=seed % 2 == 0, p_pin=0.5)
    o = oracle_epoch(s, ["fcfs", "srtf", "lpt"][seed % 3])
    h, lv, home = _kv_from_statuses(s, o)
    assert o["kv_hint"].tolist() == h.tolist()
    assert o["kv_level"].tolist() == lv.tolist()
    assert o["kv_home"].tolist() == home.tolist()


def test_kv_hints_c2_c4_grouped_route():
    for s in (c2(1), c4()):
        o = oracle_epoch(s, "srtf")
        h, lv, home = _kv_from_statuses(s, o)
        assert np.array_equal(o["kv_hint"], h) and np.array_equal(o["kv_level"], lv)
        assert np.array_equal(o["kv_home"], home)
        if s.n_futures == 1 << 17:
            assert set(np.unique(h)) == {KV_NONE, KV_RETAIN, KV_OFFLOAD, KV_DROP}


# --------------------------------------------------------------------------
# O10 resource reassignment (NEXT-2)
# --------------------------------------------------------------------------
def test_reassign_hand_derived():
    """Types 0, 1, 2 with two instances each (cap 4).  Type 0: loads (4, 3)
    plus two deferred futures -> busy 9 / cap 8 (112%) hot.  Type 1: loads
    (1, 0) -> 12.5% cold; kill its least-loaded instance 3.  Type 2: loads
    (2, 2) -> 50% neither."""
    tb = TableBuilder(i_type=[0, 0, 1, 1, 2, 2], i_cap=[4] * 6, i_base_load=[4, 3, 1, 0, 2, 2],
                      t_affinity=[AFF_NONE, AFF_NONE, AFF_NONE])
    tb.add_workflow(1, 0, [(PENDING, 0, 0, -1, -1, []), (PENDING, 0, 0, -1, -1, [])])
    s = tb.build()
    o = oracle_epoch(s, "fcfs", reassign={"u_hi_pct": 80, "u_lo_pct": 30})
    assert o["status"].tolist() == [S_ASG, S_DEF]          # instance 1 has one slot left
    assert o["t_busy"].tolist() == [9, 1, 4] and o["t_cap"].tolist() == [8, 8, 8]
    assert o["ra_kill"].tolist() == [3] and o["ra_prov"].tolist() == [0]
    # directives: type 1 at its floor, or type 0 at its ceiling -> nothing
    o = oracle_epoch(s, "fcfs", reassign={"t_min_inst": [0, 2, 0], "u_hi_pct": 80, "u_lo_pct": 30})
    assert o["ra_kill"].tolist() == []
    o = oracle_epoch(s, "fcfs", reassign={"t_max_inst": [2, 9, 9], "u_hi_pct": 80, "u_lo_pct": 30})
    assert o["ra_kill"].tolist() == []
    # balanced thresholds -> no commands ("balanced utilization")
    o = oracle_epoch(s, "fcfs", reassign={"u_hi_pct": 200, "u_lo_pct": 0})
    assert o["ra_kill"].tolist() == []


def _reassign_fraction_route(s, o, mn, mx, hi, lo):
    """O10 by another route: exact Fractions and Python sorting."""
    from fractions import Fraction
    T, I = s.n_types, s.n_instances
    busy = [0] * T
    cap = [0] * T
    cnt = [0] * T
    for i in range(I):
        t = int(s.i_type[i])
        busy[t] += int(o["i_load"][i]) + int(o["i_assigned"][i])
        cap[t] += int(s.i_cap[i])
        cnt[t] += 1
    for f in np.nonzero(o["status"] == S_DEF)[0]:
        busy[int(s.f_type[f])] += 1
    inf = Fraction(10 ** 30)
    util = [(Fraction(busy[t], cap[t]) if cap[t] else (inf if busy[t] else Fraction(0))) for t in range(T)]
    hot = [t for t in range(T) if cnt[t] < mx[t] and util[t] > Fraction(hi, 100)]
    cold = [t for t in range(T) if t not in hot and cnt[t] > mn[t] and util[t] < Fraction(lo, 100)]
    hot.sort(key=lambda t: (-util[t], t))
    cold.sort(key=lambda t: (util[t], t))
    kill, prov = [], []
    for a, b in zip(hot, cold):
        cands = [i for i in range(I) if s.i_type[i] == b]
        kill.append(min(cands, key=lambda i: (int(o["i_load"][i]) + int(o["i_assigned"][i]), -i)))
        prov.append(a)
    return busy, cap, kill, prov


@pytest.mark.parametrize("seed", range(120))
def test_reassign_fraction_route(seed):
    rng = np.random.default_rng(seed)
    s = random_table(seed, n_workflows=2 + seed % 5, max_rows=4 + seed % 20, n_types=1 + seed % 5,
                     inst_per_type=(0, 1 + seed % 4), consistent=seed % 2 == 1, max_cap=1 + seed % 7,
                     max_base=seed % 9)
    T = s.n_types
    mn = rng.integers(0, 3, T).tolist()
    mx = rng.integers(1, 6, T).tolist()
    hi, lo = int(rng.integers(30, 120)), int(rng.integers(0, 50))
    lo = min(lo, hi)
    o = oracle_epoch(s, "srtf", reassign={"t_min_inst": mn, "t_max_inst": mx, "u_hi_pct": hi,
                                          "u_lo_pct": lo})
    busy, cap, kill, prov = _reassign_fraction_route(s, o, mn, mx, hi, lo)
    assert o["t_busy"].tolist() == busy and o["t_cap"].tolist() == cap
    assert o["ra_kill"].tolist() == kill and o["ra_prov"].tolist() == prov


def test_reassign_c4_shifts_toward_hot_types():
    """with skewed demand the commands move instances toward the hot type."""
    s = c4()
    o = oracle_epoch(s, "srtf", reassign={"u_hi_pct": 80, "u_lo_pct": 30})
    busy, cap, kill, prov = _reassign_fraction_route(s, o, [0] * 8, [0xFFFF] * 8, 80, 30)
    assert o["ra_kill"].tolist() == kill and o["ra_prov"].tolist() == prov and len(kill) >= 1
    for k, p in zip(kill, prov):
        assert busy[p] * cap[s.i_type[k]] > busy[s.i_type[k]] * cap[p]    # from colder to hotter


# --------------------------------------------------------------------------
# O11 head-of-line-blocking migration (NEXT-1)
# --------------------------------------------------------------------------
def _hol_table(q, n_targets=1, target_base=0, src_base=0, aff=AFF_NONE, extra=None):
    """Type 0 instances: 0 = the blocked source, 1.. = targets.  q QUEUED
    futures at instance 0 (one per workflow), plus src_base / target_base load."""
    I = 1 + n_targets
    tb = TableBuilder(i_type=[0] * I, i_cap=[64] * I, i_base_load=[src_base] + [target_base] * n_targets,
                      t_affinity=[aff])
    for k in range(q):
        tb.add_workflow(k + 1, 0, [(QUEUED, 0, 0, 0, -1, [])] + (extra or []))
    return tb.build()


def _mig(s, theta_wait=5, theta_head=5, delta=2, age=10, head=None):
    head = head if head is not None else [10] + [0] * (s.n_instances - 1)
    return oracle_epoch(s, "fcfs", migrate={"f_age": np.full(s.n_futures, age, np.uint32),
                                            "i_head_rem": np.asarray(head, np.uint32),
                                            "theta_wait": theta_wait, "theta_head": theta_head,
                                            "delta": delta})


def test_hol_spec_examples():
    # all queues empty -> no commands
    tb = TableBuilder(i_type=[0, 0], i_cap=[4, 4], i_base_load=[0, 0], t_affinity=[AFF_NONE])
    tb.add_workflow(1, 0, [(RESOLVED, 0, 0, -1, -1, [])])
    assert _mig(tb.build())["n_migrated"] == 0
    # one instance blocked by a long head job, an idle peer -> the blocked
    # futures migrate to the idle peer: backlog 3 vs 0, delta 2:
    # moves while (moved) + 2 <= 3 - (moved) -> 1 move
    o = _mig(_hol_table(3))
    assert o["migrate_to"].tolist() == [1, -1, -1] and o["n_migrated"] == 1
    # two equally loaded instances -> no migration, the margin is unmet
    o = _mig(_hol_table(2, target_base=2))
    assert o["n_migrated"] == 0
    # not blocked (head job short) or not waiting long -> nothing
    assert _mig(_hol_table(6), head=[3, 0])["n_migrated"] == 0
    assert _mig(_hol_table(6), age=4)["n_migrated"] == 0


@pytest.mark.parametrize("q,base,delta,nt", [(q, b, d, nt) for q in (1, 4, 9, 17) for b in (0, 3)
                                              for d in (0, 1, 2, 5) for nt in (1, 2, 3)])
def test_hol_closed_form(q, base, delta, nt):
    """One source with backlog B = q (+ its base), nt idle targets at base b:
    the j-th move (j = 0, 1, ...) lands on the target level b + floor(j / nt)
    (fill from below, ties to the lowest id) and happens iff
    b + floor(j / nt) + delta <= B - j; moves stop at the first failure."""
    s = _hol_table(q, n_targets=nt, target_base=base)
    o = _mig(s, delta=delta)
    B = q
    m = 0
    while m < q and base + m // nt + delta <= B - m:
        m += 1
    assert o["n_migrated"] == m
    assert o["migrate_to"].tolist() == [1 + (j % nt) for j in range(m)] + [-1] * (q - m)
    assert o["i_mig_out"].tolist()[0] == m


def test_hol_directives():
    # STATEFUL futures never move (in-order per session)
    assert _mig(_hol_table(6, aff=AFF_STATEFUL))["n_migrated"] == 0
    # a SESSION future moves only as its session's only queued future ...
    assert _mig(_hol_table(6, aff=AFF_SESSION))["n_migrated"] == 3
    # ... and not while the session has a running future ("deferred")
    s = _hol_table(6, aff=AFF_SESSION, extra=[(RUNNING, 0, 0, 1, -1, [])])
    assert _mig(s)["n_migrated"] == 0
    # ... nor when it has a second queued future
    s = _hol_table(6, aff=AFF_SESSION, extra=[(QUEUED, 0, 0, 0, -1, [])])
    assert _mig(s)["n_migrated"] == 0


@pytest.mark.parametrize("seed", range(150))
def test_hol_invariants_random(seed):
    """Validity of every move and maximality of the greedy (a candidate left
    in place could not move even against the final backlogs)."""
    rng = np.random.default_rng(seed)
    s = random_table(seed, n_workflows=3 + seed % 6, max_rows=4 + seed % 20, n_types=1 + seed % 3,
                     inst_per_type=(1, 2 + seed % 4), consistent=True, max_cap=2 + seed % 8,
                     max_base=seed % 6)
    age = rng.integers(0, 20, s.n_futures).astype(np.uint32)
    head = rng.integers(0, 20, s.n_instances).astype(np.uint32)
    tw, th, dl = int(rng.integers(0, 15)), int(rng.integers(0, 15)), int(rng.integers(0, 4))
    o = oracle_epoch(s, "srtf", migrate={"f_age": age, "i_head_rem": head, "theta_wait": tw,
                                         "theta_head": th, "delta": dl})
    blocked = head > th
    backlog = o["i_load"].astype(np.int64) + o["i_assigned"]
    mt = o["migrate_to"]
    wf = np.repeat(np.arange(s.n_workflows), np.diff(s.wf_fut_off.astype(np.int64)))
    final = backlog.copy()
    cand = np.zeros(s.n_futures, bool)
    for f in range(s.n_futures):
        if s.f_state[f] != QUEUED:
            assert mt[f] == -1
            continue
        src, ty = int(s.f_executor[f]), int(s.f_type[f])
        aff = int(s.t_affinity[ty])
        sess = (wf == wf[f]) & (s.f_type == ty)
        ok = blocked[src] and age[f] > tw and aff != AFF_STATEFUL
        if aff == AFF_SESSION:
            ok = ok and int((sess & (s.f_state == QUEUED)).sum()) == 1 and not (sess & (s.f_state == RUNNING)).any()
        cand[f] = ok
        if mt[f] >= 0:
            assert ok and s.i_type[mt[f]] == ty and not blocked[mt[f]] and mt[f] != src
            final[src] -= 1
            final[mt[f]] += 1
    assert np.array_equal(np.bincount(mt[mt >= 0], minlength=s.n_instances), o["i_mig_in"])
    for f in np.nonzero(cand & (mt < 0))[0]:
        ty = int(s.f_type[f])
        tg = [i for i in range(s.n_instances) if s.i_type[i] == ty and not blocked[i]]
        if tg:
            assert min(final[i] for i in tg) + dl > final[int(s.f_executor[f])]


# --------------------------------------------------------------------------
# O12 batch coalescing (NEXT-4)
# --------------------------------------------------------------------------
def test_batch_spec_example():
    """batchable, max_batch = 2, three identical-method futures ->
    a batch of 2, then a batch of 1 -- in priority order (levels 9, 5, 7)."""
    tb = TableBuilder(i_type=[0], i_cap=[8], i_base_load=[0], t_affinity=[AFF_NONE])
    for k, prio in enumerate((5, 9, 7)):
        tb.add_workflow(k + 1, prio, [(PENDING, 0, 0, -1, -1, [])])
    s = tb.build()
    o = oracle_epoch(s, "fcfs", batch={"t_max_batch": [2]})
    assert o["status"].tolist() == [S_ASG] * 3
    assert o["batch_head"].tolist() == [0, 1, 1] and o["n_batches"] == 2
    # methods are separate batch keys: methods (0, 1, 0) -> rows 1 alone
    o = oracle_epoch(s, "fcfs", batch={"t_max_batch": [2], "f_method": [0, 1, 0]})
    assert o["batch_head"].tolist() == [2, 1, 2] and o["n_batches"] == 2
    # not batchable -> nothing
    o = oracle_epoch(s, "fcfs", batch={"t_max_batch": [1]})
    assert o["batch_head"].tolist() == [-1, -1, -1] and o["n_batches"] == 0


def test_batch_managed_state_rejected():
    """managed state cannot be combined with batchable agents."""
    with pytest.raises(ValueError):
        oracle_epoch(c1(), "srtf", batch={"t_max_batch": [4, 0]})     # type 0 is SESSION


@pytest.mark.parametrize("seed", range(120))
def test_batch_properties_random(seed):
    """Every batch: one instance, one method, size <= max_batch, contiguous in
    the O4 order of its (instance, method) group, headed by its first member;
    all but the group's last batch are full; unassigned futures are unbatched."""
    rng = np.random.default_rng(seed)
    s = random_table(seed, n_workflows=3 + seed % 6, max_rows=4 + seed % 20, n_types=1 + seed % 3,
                     inst_per_type=(1, 3), consistent=seed % 2 == 0, max_cap=2 + seed % 9)
    s.t_affinity[:] = AFF_NONE
    mb = rng.integers(0, 5, s.n_types)
    meth = rng.integers(0, 3, s.n_futures)
    o = oracle_epoch(s, ["fcfs", "srtf", "lpt"][seed % 3], batch={"t_max_batch": mb, "f_method": meth})
    bh = o["batch_head"]
    asg = o["status"] == S_ASG
    inst = o["instance"]
    assert (bh[~asg] == -1).all()
    nb = 0
    for i in range(s.n_instances):
        m_b = int(mb[s.i_type[i]])
        for m in range(3):
            grp = [f for f in range(s.n_futures) if asg[f] and inst[f] == i and meth[f] == m]
            if m_b <= 1:
                assert all(bh[f] == -1 for f in grp)
                continue
            grp.sort(key=lambda f: (-int(o["level"][f]), f))      # the O4 order
            for k, f in enumerate(grp):
                assert bh[f] == grp[k - k % m_b]
            nb += (len(grp) + m_b - 1) // m_b
    assert o["n_batches"] == nb
