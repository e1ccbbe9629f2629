"""Pair-key sort timing: python tools/sort_bench.py M N  (sort_path 0 onesweep / 1 classic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_0904_3151_b200 import _native, engine  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda").manual_seed(0)
i = torch.randint(0, n, (m,), device="cuda", generator=g, dtype=torch.int64)
j = torch.randint(0, n, (m,), device="cuda", generator=g, dtype=torch.int64)
keys = (i << 32) | j
del i, j
ref = None
npass = 2 * -(-max(1, (n - 1).bit_length()) // 8)
for path in (0, 1):
    with _native.options(sort_path=path):
        ts = []
        for it in range(4):
            u = keys.clone()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            engine.sort_pair_keys(u, n)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ok = True
        if ref is None:
            ref = u
        else:
            ok = bool(torch.equal(ref, u))
        ms = min(ts[1:])
        print(f"m={m} n={n} path={path} ms={ms:.3f} passes={npass} "
              f"GB/s={npass * 16 * m / ms / 1e6:.0f} same={ok}", flush=True)
        del u
