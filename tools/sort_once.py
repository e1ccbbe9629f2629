"""Sort 2.5M random pair keys once (ncu target for the onesweep sort)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0904_3151_b200 import engine  # noqa: E402

m, n = int(os.environ.get("M", 2_480_000)), 1_600_000
rng = np.random.default_rng(0)
keys = (rng.integers(0, n, m).astype(np.int64) << 32) | rng.integers(0, n, m)
t = torch.from_numpy(keys).cuda()
for _ in range(3):
    u = t.clone()
    engine.sort_pair_keys(u, n)
torch.cuda.synchronize()
print("ok", bool((u.cpu().numpy() == np.sort(keys)).all()))
