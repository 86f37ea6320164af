"""C4 epoch (4 seeds) under partition knobs, one process per setting
(SWEEP_RECIPE=survey: SURVEY 8(d)'s generator recipe):
NALAR_CUT_NEAREST, NALAR_LONG_WEIGHT, NALAR_DEEP_ALONE.  python scripts/part_sweep.py"""
import os
import subprocess
import sys

code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from nalar_gen import swe_table
from paper_2601_05109_b200 import nalar
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = []
for seed in (1, 2, 3, 4):
    s = swe_table(1 << 17, seed, recipe=os.environ.get("SWEEP_RECIPE", "default"))
    ctx = nalar.Context.for_snapshot(s); ctx.upload(s)
    st = torch.cuda.ExternalStream(ctx.stream); ev = []
    with torch.cuda.stream(st):
        for i in range(210):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); ctx.epoch("srtf"); b.record(st); ev.append((a, b))
    torch.cuda.synchronize(); ctx.close()
    out.append(round(float(np.mean([x.elapsed_time(y) for x, y in ev[10:]])) * 1e3, 2))
print(out, round(sum(out) / len(out), 2))
'''
settings = [{}] + [{"NALAR_LONG_WEIGHT": w} for w in ("1.25", "1.5", "1.75", "2", "2.5", "3")] + \
    [{"NALAR_LONG_WEIGHT": w, "NALAR_DEEP_ALONE": d} for w in ("1.5", "2") for d in ("0", "24")] + [{}]
if len(sys.argv) > 1:
    settings = [dict(kv.split("=") for kv in a.split(",")) if a != "-" else {} for a in sys.argv[1:]]
for st in settings:
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **st}, capture_output=True, text=True)
    print(st, r.stdout.strip() or r.stderr[-300:], flush=True)
