"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic (see snapshot.py / configs.py headers).
"""
from .snapshot import (AFF_NONE, AFF_SESSION, AFF_STATEFUL, CALL_BIT, FAILED, PENDING, QUEUED,
                       RESOLVED, RUNNING, Snapshot, TableBuilder)
from .configs import CONFIGS, c1, c2, c4, c5, random_table, swe_table, C1_NAMES, hol_table, with_hol_inputs
from .dynamic import Delta, RouterSim

__all__ = ["Snapshot", "TableBuilder", "CONFIGS", "c1", "c2", "c4", "c5", "random_table",
           "swe_table", "C1_NAMES", "PENDING", "QUEUED", "RUNNING", "RESOLVED", "FAILED",
           "AFF_NONE", "AFF_SESSION", "AFF_STATEFUL", "CALL_BIT", "Delta", "RouterSim", "hol_table",
           "with_hol_inputs"]
