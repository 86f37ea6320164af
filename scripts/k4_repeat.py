"""Is K4 bound by instruction fetch?  C4 / C1 epoch with K4 launched 1, 2, 3
times (NALAR_K4_REPEAT, read at library load -- one process per setting).
  python scripts/k4_repeat.py"""
import os
import subprocess
import sys

code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from nalar_gen import c1, swe_table
from paper_2601_05109_b200 import nalar
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = []
for s in (swe_table(1 << 17, 1), c1()):
    ctx = nalar.Context.for_snapshot(s); ctx.upload(s)
    st = torch.cuda.ExternalStream(ctx.stream); ev = []
    with torch.cuda.stream(st):
        for i in range(310):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); ctx.epoch("srtf"); b.record(st); ev.append((a, b))
    torch.cuda.synchronize(); ctx.close()
    out.append(round(float(np.mean([x.elapsed_time(y) for x, y in ev[10:]])) * 1e3, 2))
print(out)
'''
for n in ("1", "2", "3"):
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "NALAR_K4_REPEAT": n},
                       capture_output=True, text=True)
    print("K4 x" + n, "C4 / C1 epoch us:", r.stdout.strip() or r.stderr[-400:], flush=True)
