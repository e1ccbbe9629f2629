"""write_edges throughput: GPU formatting (eg_format_edges) vs the
reference's per-line f-string loop, on the same edges.

    python tools/io_bench.py [--m 50000000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0904_3151_b200 as eg  # noqa: E402
from paper_0904_3151_b200 import _native, engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=50_000_000)
a = ap.parse_args()
rng = np.random.default_rng(0)
i = np.sort(rng.integers(0, 20_000_000, a.m))
keys = torch.from_numpy((i << 32) | (i + rng.integers(1, 1000, a.m))).cuda()
dist = torch.from_numpy(rng.random(a.m) * 0.02).cuda()
lib = _native.lib()
m = min(a.m, 1 << 26)
ws = engine._ws(lib.eg_format_edges_workspace(m), keys.device)
out = torch.empty(m * 44, dtype=torch.uint8, device=keys.device)
need = engine.ctypes_i64(0)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _native.check(lib.eg_format_edges(keys.data_ptr(), dist.data_ptr(), m, out.data_ptr(),
                                      out.numel(), engine.ctypes_addr(need), ws.data_ptr(),
                                      ws.numel(), engine._stream(keys.device)), "fmt")
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
path = "/tmp/eg_io_bench.txt"
t0 = time.perf_counter()
eg.write_edges(path, (keys, dist), {"nodes": 20_000_000})
t_file = time.perf_counter() - t0
size = os.path.getsize(path)
os.remove(path)
# reference loop (io.py:155-156) on a 1M-edge sample
s = 1_000_000
kk = keys[:s].cpu().numpy()
dd = dist[:s].cpu().numpy()
t0 = time.perf_counter()
lines = [f"{k >> 32} {k & 0xffffffff} {v:.9f}\n" for k, v in zip(kk.tolist(), dd.tolist())]
t_ref = (time.perf_counter() - t0) * (a.m / s)
print(f"edges {a.m}: GPU format {m / t_dev / 1e6:.0f} M lines/s ({need.value / t_dev / 1e9:.1f} GB/s "
      f"of text), write_edges to /tmp {t_file:.2f} s ({size / 1e9:.2f} GB), "
      f"reference loop (extrapolated from 1M lines) {t_ref:.1f} s")
