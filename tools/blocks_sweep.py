"""Device time of the MSM stage per forced block count (option msm_blocks).

    python tools/blocks_sweep.py --config cfg3 --blocks 6,8,10,12,auto
"""
import argparse
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0904_3151_b200 as eg  # noqa: E402
from paper_0904_3151_b200 import _native, distributed, engine  # noqa: E402
from paper_0904_3151_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--blocks", default="auto")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
cfg = CONFIGS[args.config]
params = bench.params_for(cfg, eg)
data, _ = bench.make_inputs(args.config)
dev = torch.device("cuda", 0)
if cfg.metric == "hamming":
    x = torch.from_numpy(data.view(np.int64)).to(dev).reshape(1, -1, 1)
else:
    x = torch.from_numpy(data).to(dev)


def step():
    if cfg.metric == "hamming":
        return distributed.hamming_step(x, params, 1, 0)
    return distributed.build_step(x, params, cfg.metric, 1, 0)


prof = _native.Profile()
ref = None
for b in args.blocks.split(","):
    _native.lib().eg_set_option(b"msm_blocks", 0 if b == "auto" else int(b))
    step()
    best = None
    for _ in range(args.reps):
        prof.start()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = step()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        p = prof.stop()
        ms = {k: round(v["ms"], 3) for k, v in p.items()}
        if best is None or wall < best[0]:
            best = (wall, ms)
    c = distributed.last_counts(res)
    sig = (c["candidates"], c["raw"], c["new"], c["edges"])
    ok = "" if ref is None or sig == ref else "  COUNTS DIFFER"
    ref = ref or sig
    print(f"blocks={b:>4} used={c['blocks']} wall={best[0]:.1f} ms msm_stage={best[1].get('msm_stage')} "
          f"group={best[1].get('msm_group')} spill={best[1].get('msm_spill')} "
          f"max_group={c['max_group']} plan={engine._last_plan}{ok}", flush=True)
    print("   ", best[1], flush=True)
    try:
        st = (ctypes.c_ulonglong * 8)()
        _native.lib().eg_debug_msm_stats(st, 1)
        if st[0]:
            print("    msm stats (last build window): buckets %d rows %d cand %d groups %d grouped %d pairs %d"
                  % tuple(st[:6]), flush=True)
    except AttributeError:
        pass
