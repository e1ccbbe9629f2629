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
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--nvlink-gbs", type=float, default=700.0,
                help="effective all-gather bandwidth per GPU (NVLink 5: 900 GB/s per direction)")
ap.add_argument("--coll-latency-us", type=float, default=20.0)
ap.add_argument("--opt", action="append", default=[], help="name=value for eg_set_option")
a = ap.parse_args()
for o in a.opt:
    from paper_0904_3151_b200 import _native
    k_, v_ = o.split("=")
    assert _native.lib().eg_set_option(k_.encode(), int(v_)) == 0, o
cfg = CONFIGS[a.config]
params = bench.params_for(cfg, eg)
x = torch.from_numpy(bench.make_inputs(a.config)[0]).cuda()
n = x.shape[0]
ops = distributed.DeviceOps()
full_codes, _ = engine.project_codes(x, engine.validate_rows(x), params.length, params.seed,
                                     list(range(1, params.replicates + 1)))
full_norms = engine.validate_rows(x)
torch.cuda.synchronize()
# single-GPU build in the same process (the denominator of the speed-up)
one = []
for _ in range(a.reps + 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    distributed.build_step(x, params, cfg.metric, 1, 0)
    e1.record()
    torch.cuda.synchronize()
    one.append(e0.elapsed_time(e1))
one_ms = min(one[2:])
totals, edge_counts = [], []
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
        units = distributed.my_units(params.replicates * ops.unit_count(blocks, params.mismatch),
                                     a.world, r)
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
    totals.append(sum(best))
    edge_counts.append(int(ek.numel()))
# collectives of distributed.build_step, modelled (no second GPU here): one
# all-gather of codes + norms, an 8-byte plan broadcast, one gather of the
# ranks' sorted edge runs to rank 0 and its merge rounds
W = full_codes.shape[2]
gather_bytes = (a.world - 1) / a.world * (params.replicates * n * W * 8 + n * 8)
edge_bytes = sum(edge_counts) / max(1, len(edge_counts)) * (a.world - 1) * 16
coll_ms = (gather_bytes + edge_bytes) / (a.nvlink_gbs * 1e9) * 1e3 + 3 * a.coll_latency_us / 1e3
merge_ms = 0.02 * max(1, (a.world - 1).bit_length())
crit = max(totals) + coll_ms + merge_ms
print(f"single GPU {one_ms:.3f} ms; world={a.world}: slowest rank {max(totals):.3f} ms + collectives "
      f"{coll_ms:.3f} ms ({(gather_bytes + edge_bytes) / 1e6:.1f} MB at {a.nvlink_gbs:.0f} GB/s, "
      f"3 x {a.coll_latency_us:.0f} us) + merge {merge_ms:.3f} ms = {crit:.3f} ms -> modelled speed-up "
      f"{one_ms / crit:.2f}x")
