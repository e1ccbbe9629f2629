"""MSM-stage timing on one config's codes (no projection / verify in the
timed region): python tools/msm_bench.py --config cfg3 [--iters 10]
Select a library variant with EG_LIB_PATH.  Prints ms per eg_msm_pairs
call (engine.msm_pairs: units + cross-replicate filter + compaction) and
a digest of the sorted output keys, so variants can be compared."""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0904_3151_b200 as eg  # noqa: E402
from paper_0904_3151_b200 import engine, _native  # noqa: E402
from paper_0904_3151_b200.bitpool import block_partition  # noqa: E402
from paper_0904_3151_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--blocks", type=int, default=0)
ap.add_argument("--opt", action="append", default=[], help="name=value for eg_set_option")
args = ap.parse_args()
for o in args.opt:
    k, v = o.split("=")
    assert _native.lib().eg_set_option(k.encode(), int(v)) == 0, o
cfg = CONFIGS[args.config]
params = bench.params_for(cfg, eg)
data, _ = bench.make_inputs(args.config)
dev = torch.device("cuda", 0)
if cfg.metric == "hamming":
    codes = torch.from_numpy(data.view(np.int64)).to(dev).reshape(1, -1, 1)
else:
    x = torch.from_numpy(data).to(dev)
    codes, norms, bad, _ = engine.project_rows(x, params.length, params.seed,
                                               list(range(1, params.replicates + 1)))
    del x
n = codes.shape[1]
blocks = args.blocks or engine.msm_plan(codes, params.length, params.blocks, params.mismatch)
bounds = block_partition(params.length, engine.plan_design(blocks, params.mismatch)[0])
reps, masks = engine.units_for(range(codes.shape[0]), blocks, params.mismatch)
prof = _native.Profile()
times = []
for it in range(args.iters + 2):
    torch.cuda.synchronize()
    if it == 2:
        prof.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if os.environ.get("EG_RAW_PAIRS"):
        keys, info = engine.msm_pairs(codes, params.length, bounds, params.mismatch, reps, masks)
    else:   # the build's path (balanced bit view when the plan changed the blocks)
        keys, info = engine.msm_candidates(codes, params.length, params.blocks,
                                           params.mismatch, blocks=blocks)
    e1.record()
    torch.cuda.synchronize()
    if it >= 2:
        times.append(e0.elapsed_time(e1))
p = prof.stop()
engine.sort_pair_keys(keys, n)
dig = hashlib.sha256(keys.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"{args.config} blocks={blocks} units={len(reps)} msm_ms min={min(times):.3f} "
      f"med={sorted(times)[len(times) // 2]:.3f} keys={keys.numel()} raw={info['raw']} "
      f"new={info['new']} max_group={info['max_group']} digest={dig}")
print("  classes:", {k: round(v['ms'] / len(times), 3) for k, v in p.items()})
if os.environ.get("EG_STATS"):
    import ctypes
    st = (ctypes.c_ulonglong * 16)()
    rc = _native.lib().eg_debug_msm_stats(ctypes.addressof(st), 1)
    assert rc == 0, rc
    print("  stats (all iterations):", list(st))
