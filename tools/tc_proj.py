"""Time only the projection stage on cfg3-shaped data (experiments)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0904_3151_b200 import _native, engine, workloads  # noqa: E402

n = int(os.environ.get("N", 1_600_000))
rng = np.random.default_rng(0)
x = np.abs(rng.standard_normal((n, 384), dtype=np.float32))
xd = torch.from_numpy(x).cuda()
norms = engine.validate_rows(xd)
prof = _native.Profile()
for i in range(3):
    prof.start()
    codes, fix = engine.project_codes(xd, norms, 48, 0, [1, 2, 3])
    torch.cuda.synchronize()
    p = prof.stop()
    print({k: round(v["ms"], 3) for k, v in p.items()}, "fixups", int(fix.item()), flush=True)
