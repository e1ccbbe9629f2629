"""Small builds that reach every kernel family, for compute-sanitizer:

    compute-sanitizer --tool racecheck python tools/sanitize_run.py cfg1
    compute-sanitizer --tool memcheck  python tools/sanitize_run.py cfg3_small

cfg1: n=4000 config-1 rows (projection, MSM small/medium tiers, sort,
verify, two streams); cfg3_small: n=20000 config-3 rows, 3 replicates
(cross-replicate filter); tiers: a coarse forced block count on skewed bits
(medium + spill tiers); exact: the exhaustive oracle kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_0904_3151_b200 as eg  # noqa: E402
from paper_0904_3151_b200 import _native, workloads  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
if what == "cfg1":
    x = workloads.cfg1_points(4000, clusters=40)
    g = eg.build_graph(x, eg.MsmParams(0.1, 1e-6, 32, 2, 8, 1, 0))
elif what == "cfg3_small":
    x = workloads.cfg3_points(20_000)
    g = eg.build_graph(x, eg.MsmParams(0.05, 1e-6, 48, 3, 12, 3, 0))
elif what == "tiers":
    rng = np.random.default_rng(5)
    bits = (rng.random((20_000, 48)) < 0.8).astype(np.uint8)
    pool = eg.BitStringPool.from_bits(bits).partitioned(12)
    with _native.options(msm_blocks=4):
        g = eg.enumerate_pairs(pool, 3)
elif what == "exact":
    x = workloads.cfg1_points(3000, clusters=30)
    g = eg.brute_force_cosine(x, 0.1)
    eg.brute_force_hamming(eg.BitStringPool(workloads.cfg2_words(20_000, 1_000), 64), 2)
print(what, "ok", len(g) if hasattr(g, "__len__") else g.edge_count, flush=True)
