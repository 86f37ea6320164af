"""Summarise an ncu --set full report (and a launch-list CSV) into profiles/.

  python scripts/ncu_summarize.py gpurun_out/prof_TAG.ncu-rep gpurun_out/launches_TAG.csv TAG

Writes profiles/TAG_ncu_summary.md, profiles/TAG_ncu_launches.csv and
profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py's roofline).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__shared_mem_per_block_static", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    head, units, rows = raw(rep)
    ki = head.index("Kernel Name")
    md = [f"# ncu --set full summary ({tag})", "",
          f"source: `{os.path.basename(rep)}` (ncu --set full --clock-control none --import-source on, "
          "L2 flushed by a 256 MB memset before every epoch; cold-cache, serialised replays)", ""]
    traffic = {}
    per_kernel = {}
    for r in rows:
        name = r[ki].split("(")[0].split("::")[-1]
        per_kernel.setdefault(name, []).append(r)
    for name, rs in per_kernel.items():
        md.append(f"## {name} ({len(rs)} launches captured)")
        md.append("")
        md.append("| metric | unit | " + " | ".join(f"launch {i}" for i in range(len(rs))) + " |")
        md.append("|---|---|" + "---|" * len(rs))
        for m in WANT:
            if m in head:
                j = head.index(m)
                md.append(f"| {m} | {units[j]} | " + " | ".join(r[j] for r in rs) + " |")
        stalls = []
        for j, h in enumerate(head):
            if h.startswith(STALLS) and not h.endswith("not_issued"):
                try:
                    stalls.append((float(rs[0][j]), h[len(STALLS):]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(v for v, _ in stalls) or 1.0
        md.append("")
        md.append("top warp-stall reasons (launch 0, share of samples): " +
                  ", ".join(f"{n} {v / tot * 100:.0f}%" for v, n in stalls[:6]))
        md.append("")
        try:
            jr, jw = head.index("dram__bytes_read.sum"), head.index("dram__bytes_write.sum")

            def tobytes(v, u):
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            per = [tobytes(r[jr], units[jr]) + tobytes(r[jw], units[jw]) for r in rs]
            traffic[name] = sum(per) / len(per)
        except ValueError:
            pass
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    if os.path.exists(launches):
        lines = open(launches).read().splitlines()
        start = next((i for i, l in enumerate(lines) if l.startswith('"ID"')), 0)
        open(os.path.join(ROOT, "profiles", f"{tag}_ncu_launches.csv"), "w").write(
            "\n".join(lines[start:]) + "\n")
    print("\n".join(md))
    print(traffic)


if __name__ == "__main__":
    main()
