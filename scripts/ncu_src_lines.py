"""Stall samples of one ncu source capture per source line (innermost inlined
location from nvdisasm -gi).  python scripts/ncu_src_lines.py SRC.csv DIS FUNC [--top 30]"""
import collections
import csv
import re
import sys

src, dis_path, func = sys.argv[1:4]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
cols = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) > 3 and r[0].startswith("0x")]
ia, iex, iss = cols.index("Address"), cols.index("Instructions Executed"), cols.index("Warp Stall Sampling (All Samples)")
stc = [c for c in cols if c.startswith("stall_") and "Not Issued" not in c]
base = int(data[0][ia], 16)
dis = open(dis_path).read()
dis = dis[dis.index(f".text.{func}:"):]
nxt = dis.find("\n.text.", 10)
dis = dis[:nxt] if nxt > 0 else dis
loc, fresh, al = None, True, {}
for l in dis.splitlines():
    if l.strip().startswith("//## File"):
        if fresh:
            m = re.search(r'File "([^"]+)", line (\d+)', l)
            loc = (m.group(1).split("/")[-1], int(m.group(2)))
            fresh = False
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        al[int(m.group(1), 16)] = loc
        fresh = True
tot = sum(int(r[iss] or 0) for r in data)
by = collections.defaultdict(collections.Counter)
for r in data:
    L = al.get(int(r[ia], 16) - base)
    by[L]["all"] += int(r[iss] or 0)
    by[L]["exec"] += int(r[iex] or 0)
    for c in stc:
        by[L][c] += int(r[cols.index(c)] or 0)
print("total samples", tot)
for L, c in sorted(by.items(), key=lambda kv: -kv[1]["all"])[:top]:
    reasons = ", ".join(f"{k[6:]} {v}" for k, v in c.most_common() if k.startswith("stall_") and v)[:80]
    print(f"{c['all']:5d} {100 * c['all'] / max(tot, 1):5.1f}%  exec {c['exec']:7d}  {L}  {reasons}")
