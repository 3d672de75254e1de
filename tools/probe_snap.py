"""Snap dedupe counters (-DCABS_PROFILE_SNAP): rescans and greedy-pass cycles over one c2 step."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402

dev = torch.device("cuda:0")
A = workloads.make_A("c2", device=dev)
pipe = CabsPipeline(A, A.shape[0], A.shape[1], CabsConfig(k1=50, k2=50, iters=20))
pipe.run()
torch.cuda.synchronize()
c = C.cabs_debug_counters(16)
print("rescans", c[0], "greedy cycles", c[1], "probe+ballot", c[2], "rest", c[3])
