"""Snapshot container: the live future table as structure-of-arrays (numpy).

This module holds DATA ONLY -- no readiness, depth, priority or routing
arithmetic of the method lives here.  It is the one module both the oracle
side (tests, ``oracle/``) and the CUDA side (``paper_2601_05109_b200``) read
their inputs from.

Field meanings follow the paper's problem statement:
  * futures with dependency edges, creator (CALL edge) and executor
    (PAPER.md:469-485 ``tab:future-metadata``),
  * workflow / session ids carried on every future,
  * component instances with load and capacity and per-type
    state-placement directives (PAPER.md:242-258 ``tab:hint-agent``).

Encoding (the on-the-wire format of ``include/nalar.h``'s ``nalar_snapshot``):
  f_state   u8   0 PENDING, 1 QUEUED, 2 RUNNING, 3 RESOLVED, 4 FAILED
  f_type    u8   component type index  (< T)
  f_round   u8   retry round the future was created in (LPT input)
  f_executor i16 instance the future is queued/running at, -1 none
  f_pin     i16  session home instance (state placement), -1 none
  f_edge_off u32 [N+1] CSR offsets into ``edges``
  edges     u32  bit31 = 1 for a CALL (creator) edge, 0 for a DEP edge;
                 bits 0..30 = predecessor row (same workflow, earlier row)
  wf_id     u64  workflow (session) id, strictly increasing with row order
  wf_fut_off u32 [W+1] first row of each workflow
  wf_prio   i32  set_priority value of the session
  i_type    u8   type of each instance
  i_cap     u32  concurrency capacity of each instance
  i_base_load u32 load already present at the instance outside the table
  t_affinity u8  0 NONE, 1 SESSION (managed state), 2 STATEFUL directive
"""
from __future__ import annotations

from dataclasses import dataclass, field, fields

import numpy as np

PENDING, QUEUED, RUNNING, RESOLVED, FAILED = 0, 1, 2, 3, 4
AFF_NONE, AFF_SESSION, AFF_STATEFUL = 0, 1, 2
CALL_BIT = np.uint32(1 << 31)

_DTYPES = {
    "wf_id": np.uint64, "wf_fut_off": np.uint32, "wf_prio": np.int32,
    "f_state": np.uint8, "f_type": np.uint8, "f_round": np.uint8,
    "f_executor": np.int16, "f_pin": np.int16,
    "f_edge_off": np.uint32, "edges": np.uint32,
    "i_type": np.uint8, "i_cap": np.uint32, "i_base_load": np.uint32,
    "t_affinity": np.uint8,
}


@dataclass
class Snapshot:
    wf_id: np.ndarray
    wf_fut_off: np.ndarray
    wf_prio: np.ndarray
    f_state: np.ndarray
    f_type: np.ndarray
    f_round: np.ndarray
    f_executor: np.ndarray
    f_pin: np.ndarray
    f_edge_off: np.ndarray
    edges: np.ndarray
    i_type: np.ndarray
    i_cap: np.ndarray
    i_base_load: np.ndarray
    t_affinity: np.ndarray
    global_row_base: int = 0
    name: str = field(default="snapshot")
    # optional HoL-migration inputs (NEXT-1): wait age of each QUEUED future,
    # predicted remaining time of each instance's head job (one time unit)
    f_age: np.ndarray = None
    i_head_rem: np.ndarray = None
    # optional batch-coalescing key with the agent type (NEXT-4), u8
    f_method: np.ndarray = None

    def __post_init__(self):
        for f in fields(self):
            if f.name in _DTYPES:
                v = np.ascontiguousarray(getattr(self, f.name), dtype=_DTYPES[f.name])
                setattr(self, f.name, v)
        for k, dt in (("f_age", np.uint32), ("i_head_rem", np.uint32), ("f_method", np.uint8)):
            if getattr(self, k) is not None:
                setattr(self, k, np.ascontiguousarray(getattr(self, k), dtype=dt))

    # sizes --------------------------------------------------------------
    @property
    def n_futures(self) -> int:
        return int(self.f_state.shape[0])

    @property
    def n_edges(self) -> int:
        return int(self.edges.shape[0])

    @property
    def n_workflows(self) -> int:
        return int(self.wf_id.shape[0])

    @property
    def n_instances(self) -> int:
        return int(self.i_type.shape[0])

    @property
    def n_types(self) -> int:
        return int(self.t_affinity.shape[0])

    def arrays(self) -> dict:
        return {k: getattr(self, k) for k in _DTYPES}

    def nbytes(self) -> int:
        return int(sum(a.nbytes for a in self.arrays().values()))

    def copy(self) -> "Snapshot":
        kw = {k: v.copy() for k, v in self.arrays().items()}
        return Snapshot(global_row_base=self.global_row_base, name=self.name, **kw,
                        f_age=None if self.f_age is None else self.f_age.copy(),
                        i_head_rem=None if self.i_head_rem is None else self.i_head_rem.copy(),
                        f_method=None if self.f_method is None else self.f_method.copy())

    # data-layout utilities (no method arithmetic) -------------------------
    def slice_workflows(self, w0: int, w1: int) -> "Snapshot":
        """Workflows [w0, w1) as a self-contained table; rows re-based to 0.

        Instance and type tables are replicated.  ``global_row_base`` records
        where row 0 of the slice sits in this table's (global) row order.
        """
        r0 = int(self.wf_fut_off[w0])
        r1 = int(self.wf_fut_off[w1])
        e0 = int(self.f_edge_off[r0])
        e1 = int(self.f_edge_off[r1])
        edges = self.edges[e0:e1].copy()
        rows = (edges & ~CALL_BIT) - np.uint32(r0)
        edges = (edges & CALL_BIT) | rows.astype(np.uint32)
        return Snapshot(
            wf_id=self.wf_id[w0:w1], wf_fut_off=self.wf_fut_off[w0:w1 + 1] - np.uint32(r0),
            wf_prio=self.wf_prio[w0:w1],
            f_state=self.f_state[r0:r1], f_type=self.f_type[r0:r1], f_round=self.f_round[r0:r1],
            f_executor=self.f_executor[r0:r1], f_pin=self.f_pin[r0:r1],
            f_edge_off=self.f_edge_off[r0:r1 + 1] - np.uint32(e0), edges=edges,
            i_type=self.i_type, i_cap=self.i_cap, i_base_load=self.i_base_load,
            t_affinity=self.t_affinity, global_row_base=self.global_row_base + r0,
            name=f"{self.name}[w{w0}:{w1}]",
            f_age=None if self.f_age is None else self.f_age[r0:r1],
            i_head_rem=self.i_head_rem,
            f_method=None if self.f_method is None else self.f_method[r0:r1])

    def save(self, path: str) -> None:
        np.savez(path, global_row_base=np.uint64(self.global_row_base), **self.arrays())

    @staticmethod
    def load(path: str) -> "Snapshot":
        z = np.load(path)
        kw = {k: z[k] for k in _DTYPES}
        return Snapshot(global_row_base=int(z["global_row_base"]), **kw)


class TableBuilder:
    """Append-only builder: workflows are appended whole, rows in creation order."""

    def __init__(self, i_type, i_cap, i_base_load, t_affinity, name="snapshot"):
        self.name = name
        self.i_type = np.asarray(i_type, np.uint8)
        self.i_cap = np.asarray(i_cap, np.uint32)
        self.i_base_load = np.asarray(i_base_load, np.uint32)
        self.t_affinity = np.asarray(t_affinity, np.uint8)
        self.wf_id, self.wf_prio, self.wf_off = [], [], [0]
        self.state, self.type, self.round, self.exe, self.pin = [], [], [], [], []
        self.edge_off, self.edges = [0], []

    @property
    def n_rows(self) -> int:
        return len(self.state)

    def add_workflow(self, wid: int, prio: int, rows) -> None:
        """rows: list of (state, type, round, executor, pin, [(pred_local, is_call), ...]).

        Predecessors are indices local to the workflow.
        """
        base = self.n_rows
        for (st, ty, rd, ex, pn, preds) in rows:
            self.state.append(st); self.type.append(ty); self.round.append(rd)
            self.exe.append(ex); self.pin.append(pn)
            for (p, is_call) in preds:
                self.edges.append((base + p) | ((1 << 31) if is_call else 0))
            self.edge_off.append(len(self.edges))
        self.wf_id.append(wid); self.wf_prio.append(prio); self.wf_off.append(self.n_rows)

    def build(self) -> Snapshot:
        return Snapshot(
            wf_id=np.array(self.wf_id, np.uint64), wf_fut_off=np.array(self.wf_off, np.uint32),
            wf_prio=np.array(self.wf_prio, np.int32),
            f_state=np.array(self.state, np.uint8), f_type=np.array(self.type, np.uint8),
            f_round=np.array(self.round, np.uint8), f_executor=np.array(self.exe, np.int16),
            f_pin=np.array(self.pin, np.int16), f_edge_off=np.array(self.edge_off, np.uint32),
            edges=np.array(self.edges, np.uint32), i_type=self.i_type, i_cap=self.i_cap,
            i_base_load=self.i_base_load, t_affinity=self.t_affinity, name=self.name)
