"""Where does the tensor-core accumulator deviate?  Dumps the raw fp32
accumulator (eg_debug_set_tc_dump) and reports the bad entries by tile/row/col.

    EG_TC_VER=3 N=20000 python tools/tc_dump_check.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0904_3151_b200 import _native, engine  # noqa: E402

n = int(os.environ.get("N", 20000))
dim = int(os.environ.get("DIM", 384))
length = int(os.environ.get("L", 48))
reps = int(os.environ.get("R", 3))
rng = np.random.default_rng(n + dim)
x = rng.standard_normal((n, dim)).astype(np.float32)
x[: n // 4] = np.abs(x[: n // 4])
dev = torch.device("cuda", 0)
xd = torch.from_numpy(x).to(dev)
cols = length * reps
dump = torch.zeros((n, cols), dtype=torch.float32, device=dev)
lib = _native.lib()
lib.eg_debug_set_tc_dump(dump.data_ptr())
norms = engine.validate_rows(xd)
codes, _ = engine.project_codes(xd, norms, length, 0, list(range(1, reps + 1)))
torch.cuda.synchronize()
lib.eg_debug_set_tc_dump(None)
acc = dump.cpu().numpy().astype(np.float64)
r = np.concatenate([engine.directions(length, dim, 0, h) for h in range(1, reps + 1)])
exact = x.astype(np.float64) @ r.T
scale = np.linalg.norm(x.astype(np.float64), axis=1)[:, None] * np.linalg.norm(r, axis=1)[None, :]
ratio = np.abs(acc - exact) / scale
bad = np.argwhere(ratio > 1e-4)
print("max", ratio.max(), "bad entries", len(bad))
if len(bad):
    rows = np.unique(bad[:, 0])
    print("bad rows", len(rows), "first", rows[:20], "tiles", np.unique(rows // 128)[:40])
    print("bad cols", np.unique(bad[:, 1])[:60])
    print("rows within tile", np.unique(rows % 128)[:64])
    i, j = bad[0]
    print("example", i, j, acc[i, j], exact[i, j])
if len(bad):
    # per-chunk contributions: which chunk is missing / replaced?
    nkc = (dim + 31) // 32
    for (i, j) in bad[:: max(1, len(bad) // 12)][:12]:
        contrib = np.array([x[i, c * 32:(c + 1) * 32].astype(np.float64) @ r[j, c * 32:(c + 1) * 32]
                            for c in range(nkc)])
        pref = np.cumsum(contrib)
        suff = exact[i, j] - np.concatenate([[0], pref[:-1]])
        # acc == sum of the last m chunks only? == exact minus one chunk?
        best_suffix = int(np.argmin(np.abs(suff - acc[i, j])))
        miss = int(np.argmin(np.abs(exact[i, j] - contrib - acc[i, j])))
        # replaced by the row 128 rows before/after (same CTA, previous tile = 148 tiles back)
        alt = []
        for di in (-148 * 128, -128, 128):
            ii = i + di
            if 0 <= ii < n:
                ca = np.array([x[ii, c * 32:(c + 1) * 32].astype(np.float64) @ r[j, c * 32:(c + 1) * 32]
                               for c in range(nkc)])
                alt.append((di, [int(c) for c in range(nkc)
                                 if abs(exact[i, j] - contrib[c] + ca[c] - acc[i, j]) < 1e-3 * abs(acc[i, j]) + 1e-4]))
        print(f"({i},{j}) acc={acc[i, j]:.5f} exact={exact[i, j]:.5f} suffix_from={best_suffix} "
              f"err={abs(suff[best_suffix] - acc[i, j]):.2e} miss_one={miss} "
              f"err={abs(exact[i, j] - contrib[miss] - acc[i, j]):.2e} swap={alt}")
