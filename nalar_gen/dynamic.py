"""C3: a seeded discrete-event simulation of the router workflow at 80 RPS that
emits the live future table epoch by epoch and the DELTA between epochs.

DATA GENERATION ONLY: the simulator advances time, runs futures on instances
and creates / retires futures; it never computes the method's readiness,
priority or assignment -- those decisions are handed to ``step()`` by the
caller (the oracle in tests), exactly as the controller would push them.  A
simple greedy dispatcher (``warmup``) is used only to reach steady state.

Workflow (PAPER.md:622, 671-672 router workflow): classify
(ROUTER) -> w.p. 0.9 a chat branch of k ~ U{3..8} turns, each retrieve (TOOL)
-> generate (CHAT, managed-state session), then answer (CHAT); w.p. 0.1 a
coding branch code (CODE, stateful) -> test (TOOL), retried w.p. 0.3 up to 4
rounds, then answer.  Branch futures are created only when classify resolves,
retries only when a test resolves (dynamic control flow).
Arrivals are Poisson at 80/s; one epoch = 100 ms (Q19).  Service times are
lognormal; instances run up to CONC futures at once, the rest queue FIFO.
"""
from __future__ import annotations

import heapq
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .snapshot import (AFF_NONE, AFF_SESSION, AFF_STATEFUL, FAILED, PENDING, QUEUED, RESOLVED,
                       RUNNING, Snapshot)

ROUTER, TOOL, CHAT, CODE = 0, 1, 2, 3
AFFINITY = [AFF_NONE, AFF_NONE, AFF_SESSION, AFF_STATEFUL]
I_PER = 8
N_INST = 4 * I_PER
CONC = 512          # futures an instance runs at once (batched LLM serving)
CAP = 640           # queue + running admitted by the controller
SERVICE_S = {ROUTER: 0.5, TOOL: 2.0, CHAT: 6.0, CODE: 12.0}


@dataclass
class Delta:
    flags: int = 1
    upd_wf_id: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    upd_seq: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    upd_state: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    upd_executor: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int16))
    upd_pin: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int16))
    retired_wf_id: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    app_wf_id: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    app_wf_prio: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    app_state: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    app_type: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    app_round: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    app_executor: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int16))
    app_pin: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int16))
    app_edge_off: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint32))
    app_edges: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    prio_wf_id: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    prio_value: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    inst_id: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    inst_cap: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    inst_base_load: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    n_futures_after: int = 0
    n_workflows_after: int = 0


class _Wf:
    __slots__ = ("wid", "prio", "rows", "branch", "turns", "code_round", "done", "failed")

    def __init__(self, wid, prio):
        self.wid, self.prio = wid, prio
        self.rows = []          # [state, type, round, executor, pin, preds[(seq, is_call)]]
        self.branch = None
        self.turns = 0
        self.code_round = 0
        self.done = False
        self.failed = False


class RouterSim:
    def __init__(self, seed: int = 1, rps: float = 80.0, epoch_s: float = 0.1, p_fail: float = 0.002):
        self.rng = np.random.default_rng(seed)
        self.rps, self.dt, self.p_fail = rps, epoch_s, p_fail
        self.t = 0.0
        self.next_wid = 1
        self.wfs: dict[int, _Wf] = {}
        self.home: dict[tuple[int, int], int] = {}
        self.queue = [deque() for _ in range(N_INST)]
        self.running = [0] * N_INST
        self.done_heap: list = []                 # (t_done, wid, seq, inst)
        self.i_type = np.repeat(np.arange(4), I_PER).astype(np.uint8)
        self.i_cap = np.full(N_INST, CAP, np.uint32)
        self.i_base = np.zeros(N_INST, np.uint32)
        self._new_rows: list = []                 # (wid, seq) created this step
        self._changed: dict = {}                  # (wid, seq) -> True
        self._retire: list = []

    # ------------------------------------------------------------------ table
    def snapshot(self) -> Snapshot:
        wids = sorted(self.wfs)
        st, ty, rd, ex, pn, eoff, edges, off, prio = [], [], [], [], [], [0], [], [0], []
        self.row_key = []
        for wid in wids:
            wf = self.wfs[wid]
            base = len(st)
            for seq, r in enumerate(wf.rows):
                st.append(r[0]); ty.append(r[1]); rd.append(r[2]); ex.append(r[3]); pn.append(r[4])
                for (p, is_call) in r[5]:
                    edges.append((base + p) | ((1 << 31) if is_call else 0))
                eoff.append(len(edges))
                self.row_key.append((wid, seq))
            off.append(len(st))
            prio.append(wf.prio)
        return Snapshot(wf_id=np.array(wids, np.uint64), wf_fut_off=np.array(off, np.uint32),
                        wf_prio=np.array(prio, np.int32), f_state=np.array(st, np.uint8),
                        f_type=np.array(ty, np.uint8), f_round=np.array(rd, np.uint8),
                        f_executor=np.array(ex, np.int16), f_pin=np.array(pn, np.int16),
                        f_edge_off=np.array(eoff, np.uint32), edges=np.array(edges, np.uint32),
                        i_type=self.i_type, i_cap=self.i_cap, i_base_load=self.i_base,
                        t_affinity=np.array(AFFINITY, np.uint8), name=f"C3t{self.t:.1f}")

    @property
    def n_live(self) -> int:
        return sum(len(w.rows) for w in self.wfs.values())

    # ------------------------------------------------------------ mutation
    def _add(self, wf, ty, rnd, preds):
        pin = self.home.get((wf.wid, ty), -1)
        wf.rows.append([PENDING, ty, rnd, -1, pin, preds])
        self._new_rows.append((wf.wid, len(wf.rows) - 1))
        return len(wf.rows) - 1

    def _touch(self, wid, seq):
        self._changed[(wid, seq)] = True

    def _service(self, ty):
        m = SERVICE_S[ty]
        s = 0.5
        return float(self.rng.lognormal(np.log(m) - s * s / 2, s))

    def _arrive(self):
        for _ in range(int(self.rng.poisson(self.rps * self.dt))):
            wid = self.next_wid
            self.next_wid += 1
            prio = 0 if self.rng.random() < 0.9 else int(self.rng.integers(1, 9))
            wf = _Wf(wid, prio)
            self.wfs[wid] = wf
            self._add(wf, ROUTER, 0, [])

    def _on_resolved(self, wf, seq):
        ty = wf.rows[seq][1]
        if seq == 0:                                   # classify -> branch
            if self.rng.random() < 0.9:
                wf.branch = "chat"
                k = int(self.rng.integers(3, 9))
                prev = 0
                for _ in range(k):
                    r = self._add(wf, TOOL, 0, [(prev, False)])
                    g = self._add(wf, CHAT, 0, [(r, False)] + ([(prev, False)] if prev else []))
                    prev = g
                self._add(wf, CHAT, 0, [(prev, False)])     # answer
            else:
                wf.branch = "code"
                c = self._add(wf, CODE, 0, [(0, False)])
                self._add(wf, TOOL, 0, [(c, False)])
        elif wf.branch == "code" and ty == TOOL:       # a test finished
            if wf.code_round < 3 and self.rng.random() < 0.3:
                wf.code_round += 1
                c = self._add(wf, CODE, wf.code_round, [(seq, False), (seq - 1, True)])
                self._add(wf, TOOL, wf.code_round, [(c, False)])
            else:
                self._add(wf, CHAT, 0, [(seq, False)])  # answer
        elif seq == len(wf.rows) - 1 and ty == CHAT:   # the answer
            wf.done = True

    def _place(self, wid, seq, inst, new_pin):
        wf = self.wfs[wid]
        r = wf.rows[seq]
        r[0], r[3] = QUEUED, inst
        self.queue[inst].append((wid, seq))
        if new_pin:                                    # the session home
            key = (wid, r[1])
            self.home[key] = inst
            for s2, r2 in enumerate(wf.rows):
                if r2[1] == r[1] and r2[4] != inst:
                    r2[4] = inst
                    self._touch(wid, s2)

    def _advance(self):
        t1 = self.t + self.dt
        while self.done_heap and self.done_heap[0][0] <= t1:
            _, wid, seq, inst = heapq.heappop(self.done_heap)
            self.running[inst] -= 1
            wf = self.wfs[wid]
            fail = self.rng.random() < self.p_fail
            wf.rows[seq][0] = FAILED if fail else RESOLVED
            self._touch(wid, seq)
            if fail:
                wf.failed = True
            else:
                self._on_resolved(wf, seq)
        for inst in range(N_INST):
            q = self.queue[inst]
            while q and self.running[inst] < CONC:
                wid, seq = q.popleft()
                r = self.wfs[wid].rows[seq]
                r[0] = RUNNING
                self._touch(wid, seq)
                self.running[inst] += 1
                heapq.heappush(self.done_heap, (t1 + self._service(r[1]), wid, seq, inst))
        self.t = t1

    def _retire_done(self):
        for wid in list(self.wfs):
            wf = self.wfs[wid]
            # a failed workflow is aborted once nothing of it is in flight
            if wf.done or (wf.failed and not any(r[0] in (QUEUED, RUNNING) for r in wf.rows)):
                self._retire.append(wid)
                del self.wfs[wid]
                for ty in (CHAT, CODE):
                    self.home.pop((wid, ty), None)

    # --------------------------------------------------------------- drivers
    def warmup(self, epochs: int) -> None:
        """Reach steady state with a simple greedy dispatcher (input generation
        only): ready futures in row order to their home, else the least loaded
        instance of their type with room."""
        for _ in range(epochs):
            load = [len(self.queue[i]) + self.running[i] for i in range(N_INST)]
            for wid in sorted(self.wfs):
                wf = self.wfs[wid]
                for seq, r in enumerate(wf.rows):
                    if r[0] != PENDING:
                        continue
                    if not all(wf.rows[p][0] == RESOLVED for (p, c) in r[5] if not c):
                        continue
                    ty = r[1]
                    if r[4] >= 0:
                        inst = r[4]
                    else:
                        cands = [i for i in range(ty * I_PER, (ty + 1) * I_PER)]
                        inst = min(cands, key=lambda i: (load[i], i))
                    if load[inst] >= CAP:
                        continue
                    load[inst] += 1
                    self._place(wid, seq, inst, ty in (CHAT, CODE) and r[4] < 0)
            self._advance()
            self._retire_done()
            self._arrive()
        self._new_rows.clear()
        self._changed.clear()
        self._retire.clear()
        self.refresh_keys()

    def step(self, assign_row, assign_inst, new_pin) -> Delta:
        """Push one epoch's decisions (rows of the CURRENT snapshot), advance one
        epoch, and return the delta from the current table to the next one."""
        keys = self.row_key
        # the consumer applies the assignments itself (NALAR_DELTA_APPLY_ASSIGNED);
        # every later change of an existing row is sent as an update
        self._changed.clear()
        for row, inst in zip(np.asarray(assign_row).tolist(), np.asarray(assign_inst).tolist()):
            wid, seq = keys[row]
            self._place(wid, seq, inst, bool(new_pin[row]))
        self._advance()
        self._retire_done()
        retired = set(self._retire)
        self._arrive()
        # ---- the delta
        d = Delta(flags=1)
        ups = []
        fresh = set(self._new_rows)
        for (wid, seq) in sorted(self._changed):
            if wid in retired or (wid, seq) in fresh:
                continue
            r = self.wfs[wid].rows[seq]
            ups.append((wid, seq, r[0], r[3], r[4]))
        if ups:
            d.upd_wf_id = np.array([u[0] for u in ups], np.uint64)
            d.upd_seq = np.array([u[1] for u in ups], np.uint32)
            d.upd_state = np.array([u[2] for u in ups], np.uint8)
            d.upd_executor = np.array([u[3] for u in ups], np.int16)
            d.upd_pin = np.array([u[4] for u in ups], np.int16)
        d.retired_wf_id = np.array(sorted(retired), np.uint64)
        new_rows = sorted(k for k in self._new_rows if k[0] in self.wfs)
        if new_rows:
            aw, ap, ast, aty, ard, aex, apn, aeo, aed = [], [], [], [], [], [], [], [0], []
            for (wid, seq) in new_rows:
                wf = self.wfs[wid]
                r = wf.rows[seq]
                aw.append(wid); ap.append(wf.prio); ast.append(r[0]); aty.append(r[1])
                ard.append(r[2]); aex.append(r[3]); apn.append(r[4])
                for (p, is_call) in r[5]:
                    aed.append(p | ((1 << 31) if is_call else 0))
                aeo.append(len(aed))
            d.app_wf_id = np.array(aw, np.uint64); d.app_wf_prio = np.array(ap, np.int32)
            d.app_state = np.array(ast, np.uint8); d.app_type = np.array(aty, np.uint8)
            d.app_round = np.array(ard, np.uint8); d.app_executor = np.array(aex, np.int16)
            d.app_pin = np.array(apn, np.int16); d.app_edge_off = np.array(aeo, np.uint32)
            d.app_edges = np.array(aed, np.uint32)
        self._new_rows.clear()
        self._changed.clear()
        self._retire.clear()
        d.n_futures_after = self.n_live
        d.n_workflows_after = len(self.wfs)
        self.refresh_keys()
        return d

    def refresh_keys(self) -> None:
        """(workflow id, seq) of every row of the current table, in row order."""
        self.row_key = [(wid, j) for wid in sorted(self.wfs) for j in range(len(self.wfs[wid].rows))]
