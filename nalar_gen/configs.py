"""Seeded synthetic future tables shaped like the paper's workloads.

DATA GENERATION ONLY: nothing here computes readiness, depth, priority keys or
assignments.  States are drawn as a lifecycle-consistent random cut through
each workflow (a future is made RESOLVED / in flight only when its DEP
predecessors are RESOLVED), which is a property of the *input*, not the method.

Configs (BASELINE.json ``configs``; recipe in DESIGN.md "Input recipe"):
  C1  single workflow, 24 futures, 2 types x 2 instances  (hand-built fixture)
  C2  fan-out/fan-in Financial-Analyst shape, 1K workflows, 10K futures, 4 types
      ("Financial Analyst", 16 instances)
  C4  SWE recursive shape, 2^17 futures, 8 types x 8 instances, state affinity
      (Fig 1 components PAPER.md:92)
  C5  the C4 generator run to 2^20 futures (scale-out sweep)
  random_table(): tiny random tables for pins / parity fuzzing.
"""
from __future__ import annotations

import numpy as np

from .snapshot import (AFF_NONE, AFF_SESSION, AFF_STATEFUL, FAILED, PENDING, QUEUED,
                       RESOLVED, RUNNING, Snapshot, TableBuilder)

# ----------------------------------------------------------------------------
# C1: the three-agent SWE example, 24 futures.
# Rows:  0 plan(LLM); subtask s=0..5 -> doc_s(TOOL) code_s(LLM) test_s(TOOL) at
# rows 1+3s..3+3s; 19/20 retry code'/test' of subtask 1 (round 1); 21/22 retry
# of subtask 4 (round 1); 23 aggregate(LLM).  Type 0 = LLM (SESSION affinity),
# type 1 = TOOL (no affinity).  Instances: 0,1 LLM; 2,3 TOOL; cap 2 each;
# base loads (1, 0, 2, 0).  States are hand-set so that every output status
# occurs (see tests/golden/c1_srtf.txt for the hand derivation).
# ----------------------------------------------------------------------------
LLM, TOOL = 0, 1


def c1() -> Snapshot:
    R, P, F, RUN = RESOLVED, PENDING, FAILED, RUNNING
    # (name, type, round, state, executor, [DEP preds])
    spec = [
        ("plan", LLM, 0, R, 0, []),
        ("doc0", TOOL, 0, R, 2, [0]), ("code0", LLM, 0, R, 0, [0, 1]), ("test0", TOOL, 0, RUN, 3, [2]),
        ("doc1", TOOL, 0, R, 3, [0]), ("code1", LLM, 0, R, 1, [0, 4]), ("test1", TOOL, 0, R, 2, [5]),
        ("doc2", TOOL, 0, R, 2, [0]), ("code2", LLM, 0, R, 0, [0, 7]), ("test2", TOOL, 0, P, -1, [8]),
        ("doc3", TOOL, 0, F, 3, [0]), ("code3", LLM, 0, P, -1, [0, 10]), ("test3", TOOL, 0, P, -1, [11]),
        ("doc4", TOOL, 0, R, 2, [0]), ("code4", LLM, 0, R, 1, [0, 13]), ("test4", TOOL, 0, R, 3, [14]),
        ("doc5", TOOL, 0, R, 3, [0]), ("code5", LLM, 0, R, 0, [0, 16]), ("test5", TOOL, 0, P, -1, [17]),
        ("code1r", LLM, 1, P, -1, [4, 6]), ("test1r", TOOL, 1, P, -1, [19]),
        ("code4r", LLM, 1, P, -1, [13, 15]), ("test4r", TOOL, 1, P, -1, [21]),
        ("aggregate", LLM, 0, P, -1, [3, 20, 9, 12, 22, 18]),
    ]
    tb = TableBuilder(i_type=[LLM, LLM, TOOL, TOOL], i_cap=[2, 2, 2, 2], i_base_load=[1, 0, 2, 0],
                      t_affinity=[AFF_SESSION, AFF_NONE], name="C1")
    rows = [(st, ty, rd, ex, -1, [(p, False) for p in preds]) for (_, ty, rd, st, ex, preds) in spec]
    tb.add_workflow(wid=1, prio=0, rows=rows)
    return tb.build()


C1_NAMES = ["plan", "doc0", "code0", "test0", "doc1", "code1", "test1", "doc2", "code2", "test2",
            "doc3", "code3", "test3", "doc4", "code4", "test4", "doc5", "code5", "test5",
            "code1r", "test1r", "code4r", "test4r", "aggregate"]


# ----------------------------------------------------------------------------
# lifecycle-consistent state draw for one workflow
# ----------------------------------------------------------------------------
def _draw_states(rng, deps, cut, p_fail, p_frontier, progress=None):
    """deps[j] = list of DEP preds (local).  A row whose DEP preds are all
    RESOLVED is itself done (RESOLVED, or FAILED w.p. p_fail) when it lies
    before the cut -- or, when ``progress`` is given, when its own uniform draw
    is below ``progress`` (a random topological cut: every branch advances
    independently).  Rows whose DEP preds are all RESOLVED but that are not
    done form the frontier: RUNNING / QUEUED / PENDING with probabilities
    p_frontier.  Everything else is PENDING."""
    n = len(deps)
    st = np.full(n, PENDING, np.uint8)
    u = rng.random(n)
    v = rng.random(n)
    x = rng.random(n)
    pr, pq = p_frontier[0], p_frontier[0] + p_frontier[1]
    for j in range(n):
        ok = all(st[p] == RESOLVED for p in deps[j])
        if not ok:
            continue
        done = (x[j] < progress) if progress is not None else (j < cut)
        if done:
            st[j] = FAILED if u[j] < p_fail else RESOLVED
        else:
            st[j] = RUNNING if v[j] < pr else (QUEUED if v[j] < pq else PENDING)
    return st


def _dispatch(rng, st, types, pins, i_per, load, limit):
    """Executor of every started future: its pin, else a uniform instance of its
    type.  An in-flight draw whose instance is at its dispatch limit stays
    PENDING (the controller had not dispatched it), so in-flight load never
    exceeds the limit.  Mutates st and load; returns executors."""
    exe = []
    for j in range(len(types)):
        t = types[j]
        i = pins[j] if pins[j] >= 0 else int(t * i_per + rng.integers(0, i_per))
        if st[j] in (QUEUED, RUNNING):
            if load[i] < limit[i]:
                load[i] += 1
            else:
                st[j] = PENDING
        exe.append(i if st[j] in (QUEUED, RUNNING, RESOLVED) else -1)
    return exe


def _prio(rng):
    return 0 if rng.random() < 0.9 else int(rng.integers(1, 9))


# ----------------------------------------------------------------------------
# C2: Financial Analyst fan-out/fan-in
# ----------------------------------------------------------------------------
ANALYST, STOCK, BOND, SEARCH = 0, 1, 2, 3


def c2(seed: int = 1, n_workflows: int = 1000) -> Snapshot:
    rng = np.random.default_rng(seed)
    I_PER = 4
    i_type = np.repeat(np.arange(4), I_PER)
    cap = np.full(16, 32)
    base = rng.integers(0, 17, 16)
    tb = TableBuilder(i_type=i_type, i_cap=cap, i_base_load=base,
                      t_affinity=[AFF_SESSION, AFF_NONE, AFF_NONE, AFF_NONE], name=f"C2s{seed}")
    load = base.astype(np.int64).copy()
    limit = cap - rng.integers(0, 13, 16)      # the dispatcher left some headroom
    for w in range(n_workflows):
        home = int(rng.integers(0, I_PER)) if rng.random() < 0.7 else -1   # analyst instance
        types = [ANALYST] + [1 + (j % 3) for j in range(8)] + [ANALYST]
        deps = [[]] + [[0]] * 8 + [list(range(1, 9))]
        stage = int(rng.integers(0, 5))
        st = np.full(10, PENDING, np.uint8)
        if stage == 1:
            st[0] = RUNNING
        elif stage == 2:
            st[0] = RESOLVED
            for j in range(1, 9):
                u = rng.random()
                st[j] = RESOLVED if u < 0.5 else (
                    (QUEUED if rng.random() < 0.5 else RUNNING) if u < 0.75 else PENDING)
        elif stage >= 3:
            st[:9] = RESOLVED
            if stage == 4:
                st[9] = RUNNING
        pins = [home if t == ANALYST else -1 for t in types]
        exe = _dispatch(rng, st, types, pins, I_PER, load, limit)
        rows = [(int(st[j]), types[j], 0, exe[j], pins[j], [(p, False) for p in deps[j]])
                for j in range(10)]
        tb.add_workflow(wid=w + 1, prio=_prio(rng), rows=rows)
    return tb.build()


# ----------------------------------------------------------------------------
# C4 / C5: SWE recursive workflow (components PAPER.md:92)
# ----------------------------------------------------------------------------
PLANNER, DOC, SRCH, DEV, TESTER, FETCH, RUNNER, AGGREGATOR = range(8)
C4_AFFINITY = [AFF_SESSION, AFF_NONE, AFF_NONE, AFF_SESSION, AFF_STATEFUL, AFF_NONE, AFF_NONE,
               AFF_NONE]
_ZIPF = np.array([1.0 / (k ** 1.1) for k in range(1, 9)])
_ZIPF = _ZIPF / _ZIPF.sum()


def _swe_workflow(rng, deep, survey=False):
    """Returns (types, rounds, dep_preds, call_preds) in creation order."""
    types, rounds, deps, calls = [], [], [], []

    def add(t, r, d, c):
        types.append(t); rounds.append(min(r, 255)); deps.append(d); calls.append(c)
        return len(types) - 1

    plan = add(PLANNER, 0, [], [])
    if deep:
        S = int(rng.integers(1, 3))
        Rs = [int(rng.integers(40, 65)) for _ in range(S)]
    else:
        S = int(rng.integers(4, 13))
        # (survey: SURVEY.md 8(d) C4 as written, R = 1 + Geometric(0.3), cap 8)
        Rs = [min(8, (1 + int(rng.geometric(0.3))) if survey else int(rng.geometric(0.48))) for _ in range(S)]
    last_run = [None] * S
    last_review = [None] * S
    for r in range(max(Rs)):
        for s in range(S):
            if Rs[s] <= r:
                continue
            prev = last_run[s]
            src = plan if prev is None else prev
            ccreator = plan if prev is None else last_review[s]
            doc = add(DOC, r, [src], [ccreator] if rng.random() < 0.2 else [])
            srch = add(SRCH, r, [src], [ccreator] if rng.random() < 0.2 else [])
            code = add(DEV, r, [doc, srch] + ([prev] if prev is not None else []), [])
            review = add(TESTER, r, [code], [])
            fetch = add(FETCH, r, [review], [code] if rng.random() < 0.2 else [])
            run = add(RUNNER, r, [fetch, code], [code] if rng.random() < 0.2 else [])
            last_run[s] = run
            last_review[s] = review
    add(AGGREGATOR, 0, list(last_run), [])
    return types, rounds, deps, calls


def swe_table(n_futures: int, seed: int = 1, name: str = "C4", p_deep: float = 0.05,
              recipe: str = "default") -> Snapshot:
    """recipe "default": the parity-tested and benched generator (DESIGN.md 6:
    base_load U{0..4}, rounds Geometric(0.48)); "survey": SURVEY.md 8(d)'s C4
    as written (base_load U{0..16}, rounds 1 + Geometric(0.3), both cap 8)."""
    assert recipe in ("default", "survey")
    survey = recipe == "survey"
    rng = np.random.default_rng(seed)
    n_inst = 64
    i_type = np.repeat(np.arange(8), 8)
    cap = np.full(n_inst, 16)
    base = rng.integers(0, 17 if survey else 5, n_inst)
    tb = TableBuilder(i_type=i_type, i_cap=cap, i_base_load=base, t_affinity=C4_AFFINITY,
                      name=f"{name}s{seed}")
    load = base.astype(np.int64).copy()
    limit = cap - rng.integers(0, 9, n_inst)   # the dispatcher left some headroom
    wid = 0
    while tb.n_rows < n_futures:
        wid += 1
        deep = rng.random() < p_deep
        types, rounds, deps, calls = _swe_workflow(rng, deep, survey)
        n = len(types)
        left = n_futures - tb.n_rows
        if n > left:                      # truncate the last workflow to a row prefix
            n = left
            types, rounds, deps, calls = types[:n], rounds[:n], deps[:n], calls[:n]
        st = _draw_states(rng, deps, 0, p_fail=0.005, p_frontier=(0.3, 0.3),
                          progress=float(rng.uniform(0.75, 1.0)))
        homes = {}
        for t in range(8):
            if C4_AFFINITY[t] != AFF_NONE and rng.random() < 0.7:
                homes[t] = t * 8 + int(rng.choice(8, p=_ZIPF))
        pins = [homes.get(t, -1) for t in types]
        exe = _dispatch(rng, st, types, pins, 8, load, limit)
        rows = [(int(st[j]), types[j], rounds[j], exe[j], pins[j],
                 [(p, False) for p in deps[j]] + [(p, True) for p in calls[j]]) for j in range(n)]
        tb.add_workflow(wid=wid, prio=_prio(rng), rows=rows)
    return tb.build()


def c4(seed: int = 1) -> Snapshot:
    return swe_table(1 << 17, seed, "C4")


def c5(seed: int = 1, n_futures: int = 1 << 20) -> Snapshot:
    return swe_table(n_futures, seed, "C5")


# ----------------------------------------------------------------------------
# random tiny tables (fuzzing / pins)
# ----------------------------------------------------------------------------
def random_table(seed: int, n_workflows: int = 3, max_rows: int = 8, n_types: int = 2,
                 inst_per_type=(0, 3), max_preds: int = 3, p_call: float = 0.25,
                 consistent: bool = False, max_cap: int = 3, max_base: int = 3,
                 prio_range=(-3, 6), max_round: int = 3, p_pin: float = 0.4,
                 name: str = "rand") -> Snapshot:
    """Small random table.  ``consistent`` draws lifecycle-consistent states;
    otherwise states are arbitrary (any assignment is a valid input)."""
    rng = np.random.default_rng(seed)
    ipt = [int(rng.integers(inst_per_type[0], inst_per_type[1] + 1)) for _ in range(n_types)]
    if sum(ipt) == 0:
        ipt[0] = 1
    i_type = np.concatenate([np.full(k, t) for t, k in enumerate(ipt)]).astype(np.uint8)
    perm = rng.permutation(len(i_type))           # instance ids not grouped by type
    i_type = i_type[perm]
    n_inst = len(i_type)
    inst_of = {t: [i for i in range(n_inst) if i_type[i] == t] for t in range(n_types)}
    tb = TableBuilder(i_type=i_type, i_cap=rng.integers(0, max_cap + 1, n_inst),
                      i_base_load=rng.integers(0, max_base + 1, n_inst),
                      t_affinity=rng.integers(0, 3, n_types), name=f"{name}{seed}")
    wid = int(rng.integers(0, 5))
    for w in range(n_workflows):
        wid += int(rng.integers(1, 4))
        n = int(rng.integers(0, max_rows + 1))
        types = [int(rng.integers(0, n_types)) for _ in range(n)]
        deps, calls = [], []
        for j in range(n):
            k = int(rng.integers(0, min(j, max_preds) + 1))
            ps = list(rng.choice(j, size=k, replace=True)) if k else []
            d, c = [], []
            for p in ps:
                (c if rng.random() < p_call else d).append(int(p))
            deps.append(d); calls.append(c)
        if consistent:
            st = _draw_states(rng, deps, int(rng.integers(0, n + 1)), 0.15, (0.25, 0.25))
        else:
            st = rng.integers(0, 5, n).astype(np.uint8)
        homes = {}
        for t in range(n_types):
            if inst_of[t] and rng.random() < p_pin:
                homes[t] = int(rng.choice(inst_of[t]))
        rows = []
        for j in range(n):
            t = types[j]
            s = int(st[j])
            if s in (QUEUED, RUNNING) and not inst_of[t]:
                s = PENDING
            pin = homes.get(t, -1) if rng.random() < 0.85 else -1
            ex = -1
            if s in (QUEUED, RUNNING):
                ex = pin if (pin >= 0 and rng.random() < 0.7) else int(rng.choice(inst_of[t]))
            preds = [(p, False) for p in deps[j]] + [(p, True) for p in calls[j]]
            rows.append((s, t, int(rng.integers(0, max_round + 1)), ex, pin, preds))
        tb.add_workflow(wid=wid, prio=int(rng.integers(prio_range[0], prio_range[1] + 1)),
                        rows=rows)
    return tb.build()


CONFIGS = {"C1": lambda seed=1: c1(), "C2": c2, "C4": c4, "C5": c5}


# ----------------------------------------------------------------------------
# HoL-migration inputs (NEXT-1): wait ages and head-job remaining times
# ----------------------------------------------------------------------------
def with_hol_inputs(s: Snapshot, seed: int = 1, p_blocked: float = 0.25, age_max: int = 100,
                    head_long: int = 100, head_short_max: int = 20) -> Snapshot:
    """The same table plus f_age ~ U{0..age_max} (read for QUEUED futures) and
    i_head_rem = head_long on a p_blocked share of the instances (a long job at
    the head of the queue), U{0..head_short_max} elsewhere."""
    rng = np.random.default_rng(seed + 7919)
    t = s.copy()
    t.f_age = rng.integers(0, age_max + 1, s.n_futures).astype(np.uint32)
    blocked = rng.random(s.n_instances) < p_blocked
    t.i_head_rem = np.where(blocked, head_long,
                            rng.integers(0, head_short_max + 1, s.n_instances)).astype(np.uint32)
    t.name = s.name + "+hol"
    return t


def hol_table(seed: int, n_workflows: int = 24, n_types: int = 3, inst_per_type: int = 4,
              max_rows: int = 6) -> Snapshot:
    """Small tables with many QUEUED futures piled on a few instances (skewed
    executors, uneven base loads) and the NEXT-1 inputs: the head-of-line
    scenario of PAPER.md:663.  Types cycle NONE / SESSION / STATEFUL."""
    rng = np.random.default_rng(seed)
    I = n_types * inst_per_type
    i_type = np.repeat(np.arange(n_types), inst_per_type)
    tb = TableBuilder(i_type=i_type, i_cap=rng.integers(2, 12, I), i_base_load=rng.integers(0, 5, I),
                      t_affinity=[(AFF_NONE, AFF_SESSION, AFF_STATEFUL)[t % 3] for t in range(n_types)],
                      name=f"hol{seed}")
    skew = np.array([1.0 / (k + 1) ** 1.5 for k in range(inst_per_type)])
    skew /= skew.sum()
    wid = 0
    for _ in range(n_workflows):
        wid += int(rng.integers(1, 3))
        n = int(rng.integers(1, max_rows + 1))
        rows = []
        for j in range(n):
            ty = int(rng.integers(0, n_types))
            st = int(rng.choice([PENDING, QUEUED, RUNNING, RESOLVED], p=[0.3, 0.45, 0.1, 0.15]))
            ex = ty * inst_per_type + int(rng.choice(inst_per_type, p=skew)) if st in (QUEUED, RUNNING) else -1
            pin = ex if (st in (QUEUED, RUNNING) and rng.random() < 0.3) else -1
            preds = [(int(rng.integers(0, j)), False)] if j and rng.random() < 0.5 else []
            rows.append((st, ty, 0, ex, pin, preds))
        tb.add_workflow(wid=wid, prio=int(rng.integers(0, 4)), rows=rows)
    s = tb.build()
    s.f_age = rng.integers(0, 21, s.n_futures).astype(np.uint32)
    s.i_head_rem = rng.integers(0, 21, I).astype(np.uint32)
    return s
