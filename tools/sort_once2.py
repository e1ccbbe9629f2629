import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0904_3151_b200 import _native, engine
m, n, path = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = torch.Generator(device="cuda").manual_seed(0)
keys = (torch.randint(0, n, (m,), device="cuda", generator=g) << 32) | torch.randint(0, n, (m,), device="cuda", generator=g)
with _native.options(sort_path=path):
    engine.sort_pair_keys(keys, n)
torch.cuda.synchronize()
print("ok")
