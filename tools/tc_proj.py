"""Time only the fused projection (eg_project_rows) on cfg3-shaped data.

    python tools/tc_proj.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0904_3151_b200 import _native, engine  # noqa: E402

n = int(os.environ.get("N", 1_600_000))
dim = int(os.environ.get("DIM", 384))
length = int(os.environ.get("L", 48))
reps = [int(v) for v in os.environ.get("REPS", "1,2,3").split(",")]
rng = np.random.default_rng(0)
x = np.abs(rng.standard_normal((n, dim), dtype=np.float32))
xd = torch.from_numpy(x).cuda()
prof = _native.Profile()
best = None
for i in range(5):
    prof.start()
    codes, norms, bad, fix = engine.project_rows(xd, length, 0, reps)
    torch.cuda.synchronize()
    p = prof.stop()
    ms = {k: round(v["ms"], 3) for k, v in p.items()}
    if best is None or ms.get("project", 1e9) < best.get("project", 1e9):
        best = ms
print("projection ms", best, "fixups", int(fix.item()), flush=True)
