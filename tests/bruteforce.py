"""Brute-force checkers used to PIN the oracle (tests only).

Every function here reaches its answer by a different route from the oracle's
step-by-step sweep: path enumeration, forward reachability, subset
enumeration, closed-form slot lists.  None of them calls the oracle.
"""
from __future__ import annotations

import itertools

from nalar_gen import CALL_BIT, FAILED, PENDING, RESOLVED


def preds(s, f, kind=None):
    """(pred_row, is_call) of row f; kind None = all, 'dep', 'call'."""
    out = []
    for e in range(int(s.f_edge_off[f]), int(s.f_edge_off[f + 1])):
        v = int(s.edges[e])
        is_call = bool(v & int(CALL_BIT))
        p = v & ~int(CALL_BIT)
        if kind == "dep" and is_call:
            continue
        if kind == "call" and not is_call:
            continue
        out.append((p, is_call))
    return out


def depth_by_path_enumeration(s, f):
    """Length (edges) of the longest path ending at f, by enumerating every
    path backwards to a root.  Exponential; tiny DAGs only."""
    best = 0
    stack = [(f, 0)]
    while stack:
        g, length = stack.pop()
        ps = preds(s, g)
        if not ps:
            best = max(best, length)
        for (p, _) in ps:
            stack.append((p, length + 1))
    return min(best, 65535)


def doomed_by_reachability(s):
    """Rows reachable from a FAILED row by forward DEP edges through PENDING
    rows only (the consumers a failure would be pushed to)."""
    N = s.n_futures
    succ = [[] for _ in range(N)]
    for f in range(N):
        for (p, is_call) in preds(s, f):
            if not is_call:
                succ[p].append(f)
    doomed = [False] * N
    frontier = [f for f in range(N) if s.f_state[f] == FAILED]
    seen = set()
    while frontier:
        g = frontier.pop()
        for c in succ[g]:
            if s.f_state[c] == PENDING and c not in seen:
                seen.add(c)
                doomed[c] = True
                frontier.append(c)
    return doomed


def slot_list(spares):
    """Closed form of the phase-B water-fill: slots (s, i) for 1 <= s <= spare_i
    sorted by (s desc, i asc); the k-th placed future takes slot k."""
    slots = [(sv, i) for i, sp in enumerate(spares) for sv in range(1, sp + 1)]
    slots.sort(key=lambda x: (-x[0], x[1]))
    return [i for (_, i) in slots]


def lexmax_admission(order, resource_of, capacity):
    """Brute force over all subsets: the admitted set maximising the indicator
    vector lexicographically (futures listed in priority order) subject to
    |admitted on r| <= capacity[r].  ``order`` is the list of futures in
    priority order; returns the admitted set."""
    n = len(order)
    best = None
    for bits in itertools.product([1, 0], repeat=n):   # lexicographically descending
        cnt = {}
        ok = True
        for k, b in enumerate(bits):
            if b:
                r = resource_of[order[k]]
                cnt[r] = cnt.get(r, 0) + 1
                if cnt[r] > capacity.get(r, 0):
                    ok = False
                    break
        if ok:
            best = bits
            break
    return {order[k] for k in range(n) if best[k]}
