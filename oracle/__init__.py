"""TEST INFRASTRUCTURE ONLY: the CPU oracle of the Nalar policy epoch.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(paper_2601_05109_b200) never imports it.
"""
from .oracle import build_oracle, oracle_epoch, oracle_epoch_times, oracle_validate, ORACLE_SO

__all__ = ["build_oracle", "oracle_epoch", "oracle_epoch_times", "oracle_validate", "ORACLE_SO"]
