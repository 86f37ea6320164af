"""Attribute ncu per-SASS-instruction samples / executed counts to source lines.

  python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX CUBIN FUNC [--top 40]
Reads `ncu -i --page source --print-source sass --csv` and the line table of
`nvdisasm -gi` for FUNC in CUBIN (innermost inlined location per instruction).
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre, cubin, func = sys.argv[1:5]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
# optional source regions: --region name:first-last (lines of the kernel's own file)
regions = [(a.split(":")[0], *map(int, a.split(":")[1].split("-"))) for i, a in enumerate(sys.argv)
           if i > 0 and sys.argv[i - 1] == "--region"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
cols = rows[hdr]
ia, iss, iex = cols.index("Address"), cols.index("Warp Stall Sampling (All Samples)"), cols.index("Instructions Executed")
data = [r for r in rows[hdr + 1:] if len(r) > iex and r[ia].startswith("0x")]
base = int(data[0][ia], 16)
dis = subprocess.run(["nvdisasm", "-gi", "-fun", func, cubin], capture_output=True, text=True).stdout
if not dis.strip():
    dis = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
    i0 = dis.index(f".text.{func}")
    dis = dis[i0:]
loc, fresh, addr_line = None, True, {}
for l in dis.splitlines():
    if l.strip().startswith("//## File"):
        if fresh:
            m = re.search(r'File "([^"]+)", line (\d+)', l)
            loc = (m.group(1).split("/")[-1], int(m.group(2)))
            fresh = False
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        addr_line[int(m.group(1), 16)] = loc
        fresh = True
    if l.startswith(".section") and addr_line and ".text." in l and func not in l:
        break
samp, ex = collections.Counter(), collections.Counter()
for r in data:
    off = int(r[ia], 16) - base
    ln = addr_line.get(off)
    samp[ln] += int(r[iss] or 0)
    ex[ln] += int(r[iex] or 0)
ts, te = sum(samp.values()), sum(ex.values())
print(f"total samples {ts}, warp-instructions executed {te}")
for name, a, b in regions:
    sv = sum(v for k, v in samp.items() if k and a <= k[1] <= b and k[0].endswith(".cu"))
    ev = sum(v for k, v in ex.items() if k and a <= k[1] <= b and k[0].endswith(".cu"))
    print(f"region {name:12s} lines {a}-{b}: samples {100.0 * sv / ts:5.1f}%  executed {ev:9d} ({100.0 * ev / te:5.1f}%)")
for ln, v in samp.most_common(top):
    print(f"{str(ln):40s} samples {v:7d} ({100.0 * v / ts:5.1f}%)  executed {ex[ln]:9d} ({100.0 * ex[ln] / te:5.1f}%)")
