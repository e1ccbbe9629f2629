"""Recall of the MSM build against the GPU exhaustive oracle at full scale.

    python tools/recall.py [cfg3|cfg1|cfg5s] [--n N]

Prints the brute-force time (tcgen05 screen + exact verify), the exact edge
count and measure_errors of the build (reference metric: missing ratio).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0904_3151_b200 as eg  # noqa: E402
from paper_0904_3151_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="cfg3")
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
if a.config == "cfg3":
    x = workloads.cfg3_points(a.n or 1_600_000)
    params = eg.MsmParams(epsilon=0.05, gamma=1e-6, length=48, mismatch=3, blocks=12,
                          replicates=3, seed=0)
elif a.config == "cfg1":
    x = workloads.cfg1_points(a.n or 20_000)
    params = eg.MsmParams(epsilon=0.1, gamma=1e-6, length=32, mismatch=2, blocks=8,
                          replicates=1, seed=0)
else:
    x = workloads.cfg5_points(a.n or 2_000_000, clusters=(a.n or 2_000_000) // 20)
    params = eg.MsmParams(epsilon=0.15 ** 2 / 2, gamma=1e-6, length=64, mismatch=3, blocks=16,
                          replicates=2, seed=0)
xd = torch.from_numpy(x).cuda()
g = eg.build_graph(xd, params)
eg.brute_force_cosine(xd[:4096], params.epsilon)          # warm-up (allocator, module)
torch.cuda.synchronize()
t0 = time.perf_counter()
exact = eg.brute_force_cosine(xd, params.epsilon, limit=None)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
r = eg.measure_errors(g, exact)
n = x.shape[0]
print(json.dumps({"config": a.config, "n": n, "dim": x.shape[1], "eps": params.epsilon,
                  "brute_force_s": round(dt, 3), "pairs_per_s": n * (n - 1) / 2 / dt,
                  "exact_edges": r.true_edge_count, "build_edges": len(g.edge_list),
                  "missing": r.missing_count, "false": r.false_candidate_count,
                  "missing_ratio": r.missing_ratio, "recall": 1 - r.missing_ratio,
                  "per_replicate_new": r.per_replicate}))
