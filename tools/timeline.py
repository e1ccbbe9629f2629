"""GPU timeline of one build: CUDA events around every engine call, to find
idle gaps where the device waits for the host (syncs, Python overhead).

    python tools/timeline.py --config cfg3
"""
import argparse
import functools
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_0904_3151_b200 as eg  # noqa: E402
from paper_0904_3151_b200 import _native, distributed, engine, pipeline  # noqa: E402
from paper_0904_3151_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--builds", type=int, default=3)
ap.add_argument("--quiet", action="store_true")
args = ap.parse_args()
cfg = CONFIGS[args.config]
params = bench.params_for(cfg, eg)
x = torch.from_numpy(bench.make_inputs(args.config)[0]).cuda()
marks = []


def wrap(mod, name):
    fn = getattr(mod, name)

    @functools.wraps(fn)
    def inner(*a, **k):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        r = fn(*a, **k)
        h1 = time.perf_counter()
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        marks.append((name, e0, e1, h0, h1))
        return r
    setattr(mod, name, inner)


for nm in ["row_stats_async", "project_codes", "msm_plan", "msm_pairs", "raise_bad_rows",
           "sort_pair_keys", "verify", "compact_keys"]:
    wrap(engine, nm)
pipeline.engine = engine
import gc  # noqa: E402
gc_log = []


def _gc_cb(phase, info):
    if phase == "start":
        _gc_cb.t = time.perf_counter()
    else:
        gc_log.append((info["generation"], (time.perf_counter() - _gc_cb.t) * 1e3))


gc.callbacks.append(_gc_cb)
for _ in range(3):
    distributed.build_step(x, params, cfg.metric, 1, 0)
for rep in range(args.builds):
    marks.clear()
    gc_log.clear()
    prof = _native.Profile()
    prof.start()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    s.record()
    t0 = time.perf_counter()
    distributed.build_step(x, params, cfg.metric, 1, 0)
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    torch.cuda.synchronize()
    print(f"--- build {rep}: device {s.elapsed_time(e):.3f} ms, host {(time.perf_counter() - t0) * 1e3:.3f} ms")
    pr = prof.stop()
    if gc_log:
        print("   gc:", [(g, round(ms, 2)) for g, ms in gc_log])
    if s.elapsed_time(e) >= 13.0:
        print("   classes:", {k: (round(v["ms"], 3), v["count"]) for k, v in pr.items()})
        print("   capacity hint:", dict(engine._capacity_hint))
    if args.quiet and s.elapsed_time(e) < 13.0:
        continue
    prev = s
    for name, e0, e1, h0, h1 in marks:
        print(f"  {name:16s} gap_before {prev.elapsed_time(e0):7.3f}  gpu {e0.elapsed_time(e1):7.3f}"
              f"  host_call {(h1 - h0) * 1e3:7.3f}  (host t={(h0 - t0) * 1e3:7.3f})")
        prev = e1
    print(f"  tail gap {prev.elapsed_time(e):.3f}")
