"""Run a few builds of one config on cuda:0 (profiling driver for ncu).

    python tools/run_build.py --config cfg3 --reps 2
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_0904_3151_b200 as eg  # noqa: E402
from paper_0904_3151_b200 import distributed  # noqa: E402
from paper_0904_3151_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--plan", type=int, default=0, help="force a block count / design plan code")
args = ap.parse_args()
if args.plan:
    from paper_0904_3151_b200 import _native as _nat
    assert _nat.lib().eg_set_option(b"msm_blocks", args.plan) == 0
cfg = CONFIGS[args.config]
params = bench.params_for(cfg, eg)
data, _ = bench.make_inputs(args.config)
dev = torch.device("cuda", 0)
if cfg.metric == "hamming":
    import numpy as np
    x = torch.from_numpy(data.view(np.int64)).to(dev).reshape(1, -1, 1)
else:
    x = torch.from_numpy(data).to(dev)
for i in range(args.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if cfg.metric == "hamming":
        res = distributed.hamming_step(x, params, 1, 0)
    else:
        res = distributed.build_step(x, params, cfg.metric, 1, 0)
    torch.cuda.synchronize()
    print(i, f"{(time.perf_counter() - t0) * 1e3:.1f} ms", distributed.last_counts(res), flush=True)

if os.environ.get("EG_PROFILE"):
    from paper_0904_3151_b200 import _native, engine
    prof = _native.Profile()
    for i in range(2):
        prof.start()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if cfg.metric == "hamming":
            res = distributed.hamming_step(x, params, 1, 0)
        else:
            res = distributed.build_step(x, params, cfg.metric, 1, 0)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        p = prof.stop()
        print("profiled", f"{wall:.1f} ms", {k: round(v["ms"], 3) for k, v in p.items()}, flush=True)
    if cfg.metric != "hamming":
        for i in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            engine.validate_rows(x)
            torch.cuda.synchronize()
            print("row_stats", f"{(time.perf_counter() - t0) * 1e3:.2f} ms")
