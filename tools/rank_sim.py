"""Per-rank device time of the sharded build (distributed.build_step) for
world = W, emulated on one GPU without the collectives: rank r projects its
row shard, then (standing in for the NCCL all-gather) uses the full codes,
plans, runs its units, sorts and verifies its candidates.

    python tools/rank_sim.py --world 8 [--config cfg3]
"""
import argparse
import os
import sys
import time
from math import comb

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0904_3151_b200 as eg  # noqa: E402
from paper_0904_3151_b200 import distributed, engine  # noqa: E402
from paper_0904_3151_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--config", default="cfg3")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--ranks", type=int, default=3)
a = ap.parse_args()
cfg = CONFIGS[a.config]
params = bench.params_for(cfg, eg)
x = torch.from_numpy(bench.make_inputs(a.config)[0]).cuda()
n = x.shape[0]
ops = distributed.DeviceOps()
full_codes, _ = engine.project_codes(x, engine.validate_rows(x), params.length, params.seed,
                                     list(range(1, params.replicates + 1)))
full_norms = engine.validate_rows(x)
torch.cuda.synchronize()
for r in range(min(a.world, a.ranks)):
    best = None
    for _ in range(a.reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        e[0].record()
        lo, hi, per = distributed.row_shard(n, a.world, r)
        xs = x[lo:hi]
        codes_s, norms_s, bad_s = ops.project_rows(xs, params)
        e[1].record()
        blocks = ops.plan(full_codes, params)
        e[2].record()
        units = distributed.my_units(params.replicates * comb(blocks, params.mismatch), a.world, r)
        keys, info = ops.candidates(full_codes, params, units, blocks)
        e[3].record()
        keys = ops.sort(keys, n)
        e[4].record()
        ek, ed = ops.verify(x, full_norms, keys, cfg.metric, params.epsilon)
        e[5].record()
        torch.cuda.synchronize()
        ms = [e[i].elapsed_time(e[i + 1]) for i in range(5)]
        if best is None or sum(ms) < sum(best):
            best = ms
    print(f"world={a.world} rank={r} units={len(units)} total={sum(best):.3f} ms  "
          f"project={best[0]:.3f} plan={best[1]:.3f} msm={best[2]:.3f} sort={best[3]:.3f} "
          f"verify={best[4]:.3f} edges={ek.numel()}", flush=True)
