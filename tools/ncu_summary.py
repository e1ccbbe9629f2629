"""Summarise an ncu report: SOL / occupancy / warp-state metrics per kernel
and the hottest source lines (needs -lineinfo + --import-source on).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [kernel-regex]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."

WANT = ["Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Block Limit Shared Mem",
        "Block Limit Registers", "Warp Cycles Per Issued Instruction", "No Eligible",
        "Avg. Active Threads Per Warp", "L2 Hit Rate", "L1/TEX Hit Rate", "Grid Size",
        "Block Size", "Dynamic Shared Memory Per Block"]


def run(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = det[0]
ki, mi, vi, ui, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"), h.index("ID"))
per = collections.OrderedDict()
for r in det[1:]:
    if not re.search(kre, r[ki]):
        continue
    per.setdefault((r[ii], r[ki][:70]), {})[r[mi]] = (r[vi], r[ui])
for (i, k), m in per.items():
    print(f"== [{i}] {k}")
    for w in WANT:
        if w in m:
            print(f"   {w:40s} {m[w][0]} {m[w][1]}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h = raw[0]
cols = [c for c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                    "lts__t_bytes.sum", "sm__inst_executed.sum") if c in h]
for r in raw[2:]:
    if re.search(kre, r[h.index("Kernel Name")]):
        print("   raw", r[h.index("ID")], {c: r[h.index(c)] + " " + raw[1][h.index(c)] for c in cols})

# hottest source lines (first matching kernel)
txt = run("--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
          f"regex:{kre}", "--launch-count", "1")
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
fname = ""
lines = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ni = hdr.index("Instructions Executed")
    try:
        s_ = int(r[si] or 0)
        n_ = int(r[ni] or 0)
    except (ValueError, IndexError):
        continue
    lines.append((s_, n_, f"{fname}:{r[0]}", r[1].strip()[:70]))
tot = sum(x[0] for x in lines) or 1
toti = sum(x[1] for x in lines) or 1
print(f"   source lines: {len(lines)}, stall samples {tot}, warp-instructions {toti}")
print("   top CUDA lines by stall samples (share of samples, share of instructions):")
for s_, n_, loc, src in sorted(lines, reverse=True)[:30]:
    print(f"     {100*s_/tot:5.1f}%  {100*n_/toti:5.1f}%  {loc:22s} {src}")
