"""Is a pipeline re-run on new data (eager, and graph replay) identical to a fresh pipeline?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402
from workloads import CONFIGS, make_A, scaled  # noqa: E402

C.load()
dev = torch.device("cuda:0")
cfg = scaled(CONFIGS["c2"], 3000, 2000, k1=40, k2=40, iters=8)
A1 = make_A(cfg, device=dev)
A2 = make_A(scaled(CONFIGS["c2"], 3000, 2000, k1=40, k2=40, iters=8, seed=cfg.seed + 1), device=dev)
order = ["I", "J", "C", "R", "W", "r1", "s1", "P", "Q", "cen_r", "cen_c", "lab_r", "lab_c", "cw_r", "obj_r",
         "Ib", "Jb", "r2", "U", "V", "s2", "resid_sq"]


def diff(a, b):
    out = []
    for k in order:
        x, y = a[k], b[k]
        same = torch.equal(x, y) if isinstance(x, torch.Tensor) else x == y
        if not same:
            out.append(k)
    return out


fresh = CabsPipeline(A2.clone(), cfg.m, cfg.n, CabsConfig(40, 40, 8, seed=cfg.seed))
fresh.run()
ref = fresh.results()
p = CabsPipeline(A1.clone(), cfg.m, cfg.n, CabsConfig(40, 40, 8, seed=cfg.seed))
p.run()
p.A.copy_(A2)
p.run()
print("eager reuse differs in:", diff(p.results(), ref))
s = torch.cuda.Stream()
q = CabsPipeline(A1.clone(), cfg.m, cfg.n, CabsConfig(40, 40, 8, seed=cfg.seed))
with torch.cuda.stream(s):
    q.run()
    g, _ = q.capture(stream=s)
torch.cuda.synchronize()
q.A.copy_(A2)
with torch.cuda.stream(s):
    g.replay()
torch.cuda.synchronize()
print("graph replay differs in:", diff(q.results(), ref))
q2 = CabsPipeline(A2.clone(), cfg.m, cfg.n, CabsConfig(40, 40, 8, seed=cfg.seed))
q2.run()
print("second fresh differs in:", diff(q2.results(), ref))
