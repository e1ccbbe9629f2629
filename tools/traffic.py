"""DRAM bytes per build and stage from an ncu metrics CSV of run_build.py:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --csv --log-file gpurun_out/traffic_cfg3.csv python tools/run_build.py --config cfg3 --reps 2
    python tools/traffic.py cfg3 N gpurun_out/traffic_cfg3.csv [profiles/r2_traffic.json]

Stages: msm = k_msm_* (the eg_msm_pairs call), sort = k_radix_* (the
candidate sort), verify = k_verify* + the double-payload compaction scatter,
projection = k_project_h16.  Per-launch bytes = stage total / builds (builds =
k_project_h16 launches, or k_msm_hist batches / 2 for the Hamming config).
ncu replays each kernel alone with cold caches, so these are upper bounds
of the in-situ traffic."""
import collections
import csv
import json
import os
import sys

cfg, n, path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
out = sys.argv[4] if len(sys.argv) > 4 else None
rows = [r for r in csv.reader(open(path)) if r]
hdr = None
per = collections.defaultdict(lambda: collections.defaultdict(float))
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"]
    val = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6}.get(unit, 1)
    per[(d["ID"], name)][d["Metric Name"]] = val * scale


def stage_of(name):
    if name.startswith("void eg::k_msm") or name.startswith("eg::k_msm"):
        return "msm"
    if "k_radix" in name:
        return "sort"
    if "k_verify" in name or "k_flag_scatter<double>" in name:
        return "verify"
    if "k_project_h16" in name:
        return "projection"
    return None


tot = collections.defaultdict(lambda: [0.0, 0.0, 0])
builds = 0
hist = 0
for (kid, name), m in per.items():
    if "k_project_h16" in name:
        builds += 1
    if "k_msm_hist" in name:
        hist += 1
    st = stage_of(name)
    if st:
        t = tot[st]
        t[0] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        t[1] += m.get("gpu__time_duration.sum", 0)
        t[2] += 1
builds = builds or max(1, hist // 2)
res = {st: {"dram_bytes_per_launch": v[0] / builds, "ncu_ms_per_launch": v[1] / builds / 1e6,
            "kernels_per_launch": v[2] / builds, "builds": builds, "n": n}
       for st, v in tot.items()}
print(json.dumps({cfg: res}, indent=1))
if out:
    cur = json.load(open(out)) if os.path.exists(out) else {}
    cur[cfg] = res
    json.dump(cur, open(out, "w"), indent=1, sort_keys=True)
