"""Phase stamps of the fused S5 kernel (-DCABS_PROFILE_EMBED): CTA 0 and the last CTA."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402

dev = torch.device("cuda:0")
A = workloads.make_A("c2", device=dev)
pipe = CabsPipeline(A, A.shape[0], A.shape[1], CabsConfig(k1=50, k2=50, iters=20))
pipe.run()
pipe.pilot()
pipe.embed()
torch.cuda.synchronize()
t = np.array(C.cabs_debug_counters(16), dtype=np.int64).reshape(2, 8)
names = ["start", "gemm", "bar1", "norms", "bar2", "end", "loaded"]
for w, row in zip(("CTA0", "last"), t):
    print(w, " ".join(f"{names[i]} {row[i] - t[0][0]}" for i in range(7)))
