"""Run eg_msm_pairs repeatedly on cfg3 replicate-1 codes and diff the pair sets."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_0904_3151_b200 import engine, workloads
from paper_0904_3151_b200.bitpool import block_partition
x = torch.from_numpy(workloads.cfg3_points()).cuda()
codes, norms, bad, _ = engine.project_rows(x, 48, 0, [1])
k = int(os.environ.get("K", "6"))
bounds = block_partition(48, k)
reps, masks = engine.units_for([0], k, 3)
sets = []
for it in range(4):
    keys, info = engine.msm_pairs(codes, 48, bounds, 3, reps, masks)
    ks = np.sort(keys.cpu().numpy().view(np.uint64))
    dup = int((np.diff(ks) == 0).sum())
    sets.append(ks)
    print(it, "emitted", len(ks), "dups", dup, "unique", len(np.unique(ks)), info["raw"], flush=True)
c = codes.cpu().numpy().view(np.uint64)[0, :, 0]
base = np.unique(sets[0])
for it in range(1, 4):
    u = np.unique(sets[it])
    extra = np.setdiff1d(u, base); miss = np.setdiff1d(base, u)
    print(it, "extra", len(extra), "missing", len(miss))
    for kk in list(extra[:3]) + list(miss[:3]):
        i, j = int(kk >> np.uint64(32)), int(kk & np.uint64(0xffffffff))
        print("   pair", i, j, "popcount", bin(int(c[i] ^ c[j])).count("1"))
