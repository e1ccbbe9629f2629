import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_0904_3151_b200 as eg
from paper_0904_3151_b200 import engine, distributed, _native
from paper_0904_3151_b200.workloads import CONFIGS
cfg = CONFIGS["cfg3"]; params = bench.params_for(cfg, eg)
x = torch.from_numpy(bench.make_inputs("cfg3")[0]).cuda()
marks = {}
def wrap(mod, name, key):
    fn = getattr(mod, name)
    def inner(*a, **k):
        marks[key + "_in"] = time.perf_counter()
        r = fn(*a, **k)
        marks[key + "_out"] = time.perf_counter()
        return r
    setattr(mod, name, inner)
wrap(engine, "msm_plan", "plan")
lib = _native.lib()
orig = lib.eg_msm_pairs_design
def pd(*a):
    marks["pairs_in"] = time.perf_counter()
    r = orig(*a)
    marks["pairs_out"] = time.perf_counter()
    return r
lib.eg_msm_pairs_design = pd
origx = lib.eg_xrep_filter_async
def px(*a):
    marks["xrep_in"] = time.perf_counter()
    return origx(*a)
lib.eg_xrep_filter_async = px
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    distributed.build_step(x, params, cfg.metric, 1, 0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    if it >= 3:
        print(f"build {1e3*(t1-t0):.3f} ms | plan call {1e3*(marks['plan_out']-marks['plan_in']):.3f} | plan_out -> pairs_in {1e3*(marks['pairs_in']-marks['plan_out']):.3f} | pairs call {1e3*(marks['pairs_out']-marks['pairs_in']):.3f} | pairs_out -> xrep_in {1e3*(marks['xrep_in']-marks['pairs_out']):.3f}")
