"""Objective histories of the c2 bench step: is the Lloyd assignment a fixed point before c?"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402

cfgw = workloads.CONFIGS["c2"] if hasattr(workloads, "CONFIGS") else None
dev = torch.device("cuda:0")
A = workloads.make_A("c2", device=dev)
m, n = A.shape
cfg = CabsConfig(k1=50, k2=50, iters=20)
pipe = CabsPipeline(A, m, n, cfg)
pipe.run()
torch.cuda.synchronize()
r = pipe.results()
np.set_printoptions(precision=10, linewidth=200)
for key in ("obj_r", "obj_c", "tie_r", "tie_c"):
    print(key, np.asarray(r[key]))
for key in ("obj_r", "obj_c"):
    o = np.asarray(r[key])
    same = [i for i in range(1, len(o)) if o[i] == o[i - 1]]
    print(key, "first repeat at iteration", same[0] if same else None)
