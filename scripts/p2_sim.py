"""Host simulation of K1's P2 segment algorithm (debug aid, not a test oracle):
B1 transfers per sub-segment, B2 export chain, B3 sweeps, executed
sequentially in Python on one workflow, compared with a plain sweep.

  python scripts/p2_sim.py [--n 131072] [--seed 1] [--wf W]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from nalar_gen import swe_table  # noqa: E402

MAXI = 7


def preds(s, f):
    out = []
    for e in range(int(s.f_edge_off[f]), int(s.f_edge_off[f + 1])):
        v = int(s.edges[e])
        out.append((v & 0x7FFFFFFF, (v >> 31) == 0))
    return out


def plain(s, fa, fb):
    d, dm = {}, {}
    for f in range(fa, fb):
        dd, bad = 0, False
        for p, dep in preds(s, f):
            dd = max(dd, d[p] + 1)
            if dep and (s.f_state[p] == 4 or dm[p]):
                bad = True
        d[f] = min(dd, 65535)
        dm[f] = s.f_state[f] == 0 and bad
    return d, dm


def segmented(s, fa, fb, seg=32):
    # B1: sub-segments inside each 32-row region, closed when the interface would exceed MAXI
    subs = []          # (start, end, iface list, direct)
    vec, dmask, export = {}, {}, set()
    for c0 in range(fa, fb, seg):
        c1 = min(c0 + seg, fb)
        cs, iface = c0, []
        f = c0
        while f < c1:
            ps = preds(s, f)
            outside = []
            for p, _ in ps:
                if p < cs and p not in iface and p not in outside:
                    outside.append(p)
            if len(iface) + len(outside) > MAXI and f > cs:
                subs.append((cs, f, iface, False))
                cs, iface = f, []
                continue                       # redo row f as the first of a new sub-segment
            if len(outside) > MAXI:            # a single row wider than the interface: direct
                for p, _ in ps:
                    export.add(p)
                subs.append((f, f + 1, [], True))
                cs, iface = f + 1, []
                f += 1
                continue
            for p in outside:
                iface.append(p)
                export.add(p)
            v = [None] * (MAXI + 1)
            dm = 0
            if not ps:
                v[MAXI] = 0
            for p, dep in ps:
                if p >= cs:
                    for i in range(MAXI + 1):
                        if vec[p][i] is not None:
                            v[i] = max(v[i] or 0, vec[p][i] + 1) if v[i] is not None else vec[p][i] + 1
                    if dep and s.f_state[p] == 0:
                        dm |= dmask[p]
                    if dep and s.f_state[p] == 4:
                        dm |= 0x80
                else:
                    i = iface.index(p)
                    v[i] = max(v[i], 1) if v[i] is not None else 1
                    if dep and s.f_state[p] == 0:
                        dm |= 1 << i
                    if dep and s.f_state[p] == 4:
                        dm |= 0x80
            vec[f] = v
            dmask[f] = dm if s.f_state[f] == 0 else 0
            f += 1
        if cs < c1:
            subs.append((cs, c1, iface, False))
    # B2: chain over sub-segments, exports only (direct ones: all rows swept)
    val = {}
    for (a, b, iface, direct) in subs:
        if direct:
            d, dm = 0, False
            for p, dep in preds(s, a):
                d = max(d, val[p][0] + 1)
                dm |= dep and (s.f_state[p] == 4 or val[p][1])
            val[a] = (min(d, 65535), s.f_state[a] == 0 and dm)
            continue
        for f in range(a, b):
            if f not in export:
                continue
            v = vec[f]
            d = v[MAXI] if v[MAXI] is not None else 0
            bad = 0
            for i, x in enumerate(iface):
                if v[i] is not None:
                    d = max(d, val[x][0] + v[i])
                if val[x][1]:
                    bad |= 1 << i
            val[f] = (min(d, 65535), (dmask[f] & (0x80 | bad)) != 0)
    # B3: sweep each sub-segment with exports final
    out_d, out_m = {}, {}
    for (a, b, iface, direct) in subs:
        for f in range(a, b):
            d, dm = 0, False
            for p, dep in preds(s, f):
                pv = out_d.get(p) if p >= a else val[p][0]
                pm = out_m.get(p) if p >= a else val[p][1]
                d = max(d, pv + 1)
                dm |= dep and (s.f_state[p] == 4 or pm)
            out_d[f] = min(d, 65535)
            out_m[f] = s.f_state[f] == 0 and dm
    return out_d, out_m, subs


ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 17)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--wf", type=int, default=-1)
a = ap.parse_args()
s = swe_table(a.n, a.seed)
off = s.wf_fut_off.astype(np.int64)
ws = [a.wf] if a.wf >= 0 else [w for w in range(s.n_workflows) if off[w + 1] - off[w] >= 128]
nsub, nrow, ndirect = 0, 0, 0
for w in ws:
    fa, fb = int(off[w]), int(off[w + 1])
    d0, m0 = plain(s, fa, fb)
    d1, m1, subs = segmented(s, fa, fb)
    nsub += len(subs); nrow += fb - fa; ndirect += sum(1 for x in subs if x[3])
    for f in range(fa, fb):
        assert d0[f] == d1[f] and m0[f] == m1[f], (w, f - fa, d0[f], d1[f], m0[f], m1[f])
print(f"{len(ws)} long workflows OK; {nrow} rows, {nsub} sub-segments ({nrow / max(nsub, 1):.1f} rows each), "
      f"{ndirect} direct rows")
