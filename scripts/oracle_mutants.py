"""Mutation check of the oracle pins (CPU only).

For each mutant: copy oracle/, nalar_gen/, tests/ into a scratch directory,
apply one plausible mistake to oracle/nalar_oracle.c, rebuild the oracle there
and run tests/test_oracle_pins.py.  Every mutant must make at least one pin
fail; a surviving mutant means an unpinned output.

usage: python scripts/oracle_mutants.py [name ...]
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, old, new): each `old` must occur in nalar_oracle.c exactly once
MUTANTS = [
    ("doom_not_transitive", "if (t->f_state[s] == S_FAILED || doomed[s]) dm = 1;",
     "if (t->f_state[s] == S_FAILED) dm = 1;"),
    ("call_edges_gate", "if (!is_call) {\n                if (t->f_state[s] == S_FAILED",
     "if (1) {\n                if (t->f_state[s] == S_FAILED"),
    ("depth_dep_only", "if (cand > d) d = cand;", "if (!is_call && cand > d) d = cand;"),
    ("order_reversed_tie", "return f < g ? -1 : (f > g ? 1 : 0);", "return f < g ? 1 : (f > g ? -1 : 0);"),
    ("argmax_ties_highest", "spare[i] > best_sp) { best = i;", "spare[i] >= best_sp && spare[i] > 0) { best = i;"),
    # VERDICT r1 What's weak #1(a): pinned_pending counting every pinned row
    ("pinned_pending_any_state", "if (st == S_PENDING && t->f_pin[f] != -1) a[7] += 1;",
     "if (t->f_pin[f] != -1) a[7] += 1;"),
    # VERDICT r1 What's weak #1(b): Q13 first placement = first PENDING non-doomed unpinned
    ("q13_first_pending_unpinned",
     "if (ready[f] && t->f_pin[f] == -1 && first_ready_unp[wt] < 0) first_ready_unp[wt] = f;",
     "if (st == S_PENDING && !doomed[f] && t->f_pin[f] == -1 && first_ready_unp[wt] < 0) first_ready_unp[wt] = f;"),
    # Q13 variant: the first ready future, pinned or not
    ("q13_first_ready_any_pin",
     "if (ready[f] && t->f_pin[f] == -1 && first_ready_unp[wt] < 0) first_ready_unp[wt] = f;",
     "if (ready[f] && first_ready_unp[wt] < 0) first_ready_unp[wt] = f;"),
    # Q12: stateful fence ignoring doom
    ("q12_fence_counts_doomed",
     "if (st == S_PENDING && !doomed[f] && first_pending[wt] < 0) first_pending[wt] = f;",
     "if (st == S_PENDING && first_pending[wt] < 0) first_pending[wt] = f;"),
    ("ready_count_pending", "if (ready[f]) a[2] += 1;", "if (st == S_PENDING) a[2] += 1;"),
    ("max_round_sum", "if (t->f_round[f] > a[9]) a[9] = t->f_round[f];", "a[9] += t->f_round[f];"),
    ("level_no_clamp_low", "if (lv < 0) lv = 0;", "if (lv < 0) lv = -lv;"),
    ("spare_soft", "if (spare[i] < 0) spare[i] = 0;", "if (spare[i] < 0) spare[i] = 1;"),
]


def run(name: str, old: str, new: str) -> bool:
    with tempfile.TemporaryDirectory(prefix=f"mut_{name}_") as d:
        for sub in ("oracle", "nalar_gen", "tests"):
            shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        src = os.path.join(d, "oracle", "nalar_oracle.c")
        text = open(src).read()
        assert text.count(old) == 1, (name, text.count(old))
        open(src, "w").write(text.replace(old, new))
        r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-x",
                            "-p", "no:cacheprovider"], cwd=d, capture_output=True, text=True)
        killed = r.returncode != 0
        tail = (r.stdout.strip().splitlines() or [""])[-1]
        print(f"{name:30s} {'KILLED' if killed else 'SURVIVED'}  {tail}", flush=True)
        return killed


if __name__ == "__main__":
    want = set(sys.argv[1:])
    res = [run(*m) for m in MUTANTS if not want or m[0] in want]
    sys.exit(0 if all(res) else 1)
