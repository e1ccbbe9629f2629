"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py gpurun_out/launches_cfg3.csv
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h, start = r, i
        break
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
for r in rows[start + 1:]:
    if len(r) != len(h):
        continue
    k = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("eg::", "")
    agg[k][0] += 1
    agg[k][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
tot = sum(v for _, v in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:44s} {c:8d} {v:9.3f} {100 * v / tot:5.1f}%")
print(f"{'total':44s} {sum(c for c, _ in agg.values()):8d} {tot:9.3f}")
