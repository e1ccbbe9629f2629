"""Per-source-line totals (stall samples, warp instructions, active lanes) of
one kernel launch in an ncu report (needs -lineinfo + --import-source on).

    python tools/ncu_lines.py rep.ncu-rep kernel-regex [launch-skip] [--by-instr]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else "0"
by_instr = "--by-instr" in sys.argv
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}", "--launch-skip", skip, "--launch-count",
                      "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, fname = None, ""
agg = collections.defaultdict(lambda: [0, 0, 0, ""])
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
    try:
        s_ = int(r[4] or 0)
        n_ = int(r[7] or 0)
        t_ = int(r[8] or 0)
    except (ValueError, IndexError):
        continue
    a = agg[(fname, int(r[0]))]
    a[0] += s_
    a[1] += n_
    a[2] += t_
    a[3] = r[1].strip()[:80]
tots = sum(v[0] for v in agg.values()) or 1
totn = sum(v[1] for v in agg.values()) or 1
print(f"stall samples {tots}, warp-instructions {totn}")
key = (lambda kv: kv[1][1]) if by_instr else (lambda kv: kv[1][0])
for (f, ln), (s_, n_, t_, src) in sorted(agg.items(), key=key, reverse=True)[:45]:
    act = t_ / n_ if n_ else 0
    print(f"{100*s_/tots:5.1f}% {100*n_/totn:5.1f}% act{act:5.1f} {f}:{ln:<5d} {src}")
