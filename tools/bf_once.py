"""One GPU brute-force call on cfg3-shaped rows (for ncu captures).

    N=200000 python tools/bf_once.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0904_3151_b200 as eg  # noqa: E402
from paper_0904_3151_b200 import workloads  # noqa: E402

x = torch.from_numpy(workloads.cfg3_points(int(os.environ.get("N", 200_000)))).cuda()
e = eg.brute_force_cosine(x, 0.05, limit=None)
torch.cuda.synchronize()
print("edges", len(e))
