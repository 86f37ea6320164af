"""ctypes loader for oracle/liboracle.so (TEST INFRASTRUCTURE ONLY).

Builds the C oracle with gcc -O2 (no SIMD intrinsics, no threads) on first
use.  Inputs are nalar_gen.Snapshot objects; outputs are numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SRC = os.path.join(HERE, "nalar_oracle.c")
ORACLE_SO = os.path.join(HERE, "liboracle.so")

POLICIES = {"fcfs": 0, "srtf": 1, "lpt": 2}


class _Table(C.Structure):
    _fields_ = [("n_futures", C.c_uint32), ("n_edges", C.c_uint32), ("n_workflows", C.c_uint32),
                ("n_instances", C.c_uint32), ("n_types", C.c_uint32), ("levels", C.c_uint32),
                ("wf_id", C.c_void_p), ("wf_fut_off", C.c_void_p), ("wf_prio", C.c_void_p),
                ("f_state", C.c_void_p), ("f_type", C.c_void_p), ("f_round", C.c_void_p),
                ("f_executor", C.c_void_p), ("f_pin", C.c_void_p), ("f_edge_off", C.c_void_p),
                ("edges", C.c_void_p), ("i_type", C.c_void_p), ("i_cap", C.c_void_p),
                ("i_base_load", C.c_void_p), ("t_affinity", C.c_void_p)]


class _Out(C.Structure):
    _fields_ = [("status", C.c_void_p), ("level", C.c_void_p), ("depth", C.c_void_p),
                ("instance", C.c_void_p), ("new_pin", C.c_void_p), ("wf_agg", C.c_void_p),
                ("i_load", C.c_void_p), ("i_spare", C.c_void_p), ("i_assigned", C.c_void_p),
                ("assign_row", C.c_void_p), ("assign_inst", C.c_void_p),
                ("kv_hint", C.c_void_p), ("kv_level", C.c_void_p), ("kv_home", C.c_void_p),
                ("n_assigned", C.c_uint32), ("n_ready", C.c_uint32), ("n_eligible", C.c_uint32),
                ("n_doomed", C.c_uint32)]


class _RaParams(C.Structure):
    _fields_ = [("t_min_inst", C.c_void_p), ("t_max_inst", C.c_void_p),
                ("u_hi_pct", C.c_uint32), ("u_lo_pct", C.c_uint32)]


class _RaOut(C.Structure):
    _fields_ = [("t_busy", C.c_void_p), ("t_cap", C.c_void_p), ("kill_inst", C.c_void_p),
                ("prov_type", C.c_void_p), ("n_pairs", C.c_uint32)]


class _MigParams(C.Structure):
    _fields_ = [("f_age", C.c_void_p), ("i_head_rem", C.c_void_p), ("theta_wait", C.c_uint32),
                ("theta_head", C.c_uint32), ("delta", C.c_uint32)]


class _MigOut(C.Structure):
    _fields_ = [("migrate_to", C.c_void_p), ("i_mig_in", C.c_void_p), ("i_mig_out", C.c_void_p),
                ("n_migrated", C.c_uint32)]


class _BatchParams(C.Structure):
    _fields_ = [("t_max_batch", C.c_void_p), ("f_method", C.c_void_p)]


class _BatchOut(C.Structure):
    _fields_ = [("batch_head", C.c_void_p), ("n_batches", C.c_uint32)]


_lib = None


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(ORACLE_SO) or \
            os.path.getmtime(ORACLE_SO) < os.path.getmtime(ORACLE_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", ORACLE_SO,
                               ORACLE_SRC])
    return ORACLE_SO


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        _lib = C.CDLL(ORACLE_SO)
        _lib.oracle_validate.argtypes = [C.POINTER(_Table), C.POINTER(C.c_int64)]
        _lib.oracle_epoch.argtypes = [C.POINTER(_Table), C.c_int, C.POINTER(_Out)]
        _lib.oracle_epoch_timed.argtypes = [C.POINTER(_Table), C.c_int, C.POINTER(_Out), C.c_int, C.c_void_p]
        _lib.oracle_reassign.argtypes = [C.POINTER(_Table), C.POINTER(_Out), C.POINTER(_RaParams),
                                         C.POINTER(_RaOut)]
        _lib.oracle_migrate.argtypes = [C.POINTER(_Table), C.POINTER(_Out), C.POINTER(_MigParams),
                                        C.POINTER(_MigOut)]
        _lib.oracle_batch.argtypes = [C.POINTER(_Table), C.POINTER(_Out), C.POINTER(_BatchParams),
                                      C.POINTER(_BatchOut)]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a.size else C.c_void_p(0)


def _table(s, levels):
    arrs = s.arrays()
    t = _Table(s.n_futures, s.n_edges, s.n_workflows, s.n_instances, s.n_types, levels,
               *[_ptr(arrs[k]) for k in ("wf_id", "wf_fut_off", "wf_prio", "f_state", "f_type",
                                         "f_round", "f_executor", "f_pin", "f_edge_off", "edges",
                                         "i_type", "i_cap", "i_base_load", "t_affinity")])
    return t, arrs   # keep arrays alive


def oracle_validate(s, levels: int = 256):
    lib = _load()
    t, keep = _table(s, levels)
    err = C.c_int64(-1)
    rc = lib.oracle_validate(C.byref(t), C.byref(err))
    return rc, err.value


def oracle_epoch_times(s, policy="srtf", reps: int = 5, levels: int = 256) -> np.ndarray:
    """Seconds per oracle epoch (O1-O9), timed inside C around the epoch
    function only (bench.py's cpu_baseline); outputs allocated once."""
    lib = _load()
    pol = POLICIES[policy] if isinstance(policy, str) else int(policy)
    t, keep = _table(s, levels)
    N, W, I, T = s.n_futures, s.n_workflows, s.n_instances, s.n_types
    bufs = [np.zeros(N, np.uint8), np.zeros(N, np.uint8), np.zeros(N, np.uint16), np.zeros(N, np.int16),
            np.zeros(N, np.uint8), np.zeros(W * 10, np.uint32), np.zeros(I, np.uint32), np.zeros(I, np.uint32),
            np.zeros(I, np.uint32), np.zeros(max(N, 1), np.uint32), np.zeros(max(N, 1), np.int16),
            np.zeros(W * T, np.uint8), np.zeros(W * T, np.uint8), np.zeros(W * T, np.int16)]
    o = _Out(*[_ptr(b) for b in bufs], 0, 0, 0, 0)
    ns = np.zeros(reps, np.uint64)
    if lib.oracle_epoch_timed(C.byref(t), pol, C.byref(o), reps, ns.ctypes.data_as(C.c_void_p)) != 0:
        raise ValueError("oracle: invalid table")
    return ns.astype(np.float64) * 1e-9


def oracle_epoch(s, policy="srtf", levels: int = 256, reassign=None, migrate=None, batch=None) -> dict:
    """One epoch; ``reassign`` = dict(t_min_inst, t_max_inst, u_hi_pct, u_lo_pct)
    also runs O10 (resource reassignment) on the result."""
    lib = _load()
    pol = POLICIES[policy] if isinstance(policy, str) else int(policy)
    t, keep = _table(s, levels)
    N, W, I = s.n_futures, s.n_workflows, s.n_instances
    out = {
        "status": np.zeros(N, np.uint8), "level": np.zeros(N, np.uint8),
        "depth": np.zeros(N, np.uint16), "instance": np.zeros(N, np.int16),
        "new_pin": np.zeros(N, np.uint8), "wf_agg": np.zeros((W, 10), np.uint32),
        "i_load": np.zeros(I, np.uint32), "i_spare": np.zeros(I, np.uint32),
        "i_assigned": np.zeros(I, np.uint32), "assign_row": np.zeros(max(N, 1), np.uint32),
        "assign_inst": np.zeros(max(N, 1), np.int16),
        "kv_hint": np.zeros((W, s.n_types), np.uint8), "kv_level": np.zeros((W, s.n_types), np.uint8),
        "kv_home": np.zeros((W, s.n_types), np.int16),
    }
    o = _Out(*[_ptr(out[k]) for k in ("status", "level", "depth", "instance", "new_pin", "wf_agg",
                                      "i_load", "i_spare", "i_assigned", "assign_row",
                                      "assign_inst", "kv_hint", "kv_level", "kv_home")], 0, 0, 0, 0)
    rc = lib.oracle_epoch(C.byref(t), pol, C.byref(o))
    if rc != 0:
        raise ValueError("oracle: invalid table")
    if reassign is not None:            # O10 (NEXT-2) on the finished epoch
        T = s.n_types
        mn = np.ascontiguousarray(reassign.get("t_min_inst", np.zeros(T)), np.uint16)
        mx = np.ascontiguousarray(reassign.get("t_max_inst", np.full(T, 0xFFFF)), np.uint16)
        ra = {"t_busy": np.zeros(T, np.uint32), "t_cap": np.zeros(T, np.uint32),
              "kill_inst": np.zeros(max(T, 1), np.int16), "prov_type": np.zeros(max(T, 1), np.int16)}
        prm = _RaParams(_ptr(mn), _ptr(mx), int(reassign.get("u_hi_pct", 80)),
                        int(reassign.get("u_lo_pct", 30)))
        ro = _RaOut(*[_ptr(ra[k]) for k in ("t_busy", "t_cap", "kill_inst", "prov_type")], 0)
        lib.oracle_reassign(C.byref(t), C.byref(o), C.byref(prm), C.byref(ro))
        out["t_busy"], out["t_cap"] = ra["t_busy"], ra["t_cap"]
        out["ra_kill"] = ra["kill_inst"][:ro.n_pairs].copy()
        out["ra_prov"] = ra["prov_type"][:ro.n_pairs].copy()
    if migrate is not None:             # O11 (NEXT-1) on the finished epoch
        age = np.ascontiguousarray(migrate["f_age"], np.uint32)
        head = np.ascontiguousarray(migrate["i_head_rem"], np.uint32)
        mo = {"migrate_to": np.zeros(max(N, 1), np.int16), "i_mig_in": np.zeros(max(I, 1), np.uint32),
              "i_mig_out": np.zeros(max(I, 1), np.uint32)}
        prm = _MigParams(_ptr(age), _ptr(head), int(migrate.get("theta_wait", 0)),
                         int(migrate.get("theta_head", 0)), int(migrate.get("delta", 2)))
        ro = _MigOut(*[_ptr(mo[k]) for k in ("migrate_to", "i_mig_in", "i_mig_out")], 0)
        lib.oracle_migrate(C.byref(t), C.byref(o), C.byref(prm), C.byref(ro))
        out["migrate_to"] = mo["migrate_to"][:N].copy()
        out["i_mig_in"], out["i_mig_out"] = mo["i_mig_in"][:I].copy(), mo["i_mig_out"][:I].copy()
        out["n_migrated"] = ro.n_migrated
    if batch is not None:               # O12 (NEXT-4) on the finished epoch
        mb = np.ascontiguousarray(batch["t_max_batch"], np.uint16)
        meth = batch.get("f_method")
        meth = None if meth is None else np.ascontiguousarray(meth, np.uint8)
        bh = np.zeros(max(N, 1), np.int32)
        prm = _BatchParams(_ptr(mb), _ptr(meth) if meth is not None else None)
        bo = _BatchOut(_ptr(bh), 0)
        if lib.oracle_batch(C.byref(t), C.byref(o), C.byref(prm), C.byref(bo)) != 0:
            raise ValueError("oracle: a batchable type with managed state (PAPER.md:576)")
        out["batch_head"] = bh[:N].copy()
        out["n_batches"] = bo.n_batches
    na = o.n_assigned
    out["assign_row"] = out["assign_row"][:na].copy()
    out["assign_inst"] = out["assign_inst"][:na].copy()
    out["n_ready"], out["n_eligible"], out["n_doomed"] = o.n_ready, o.n_eligible, o.n_doomed
    return out
