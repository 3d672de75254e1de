"""c3 k-means pair timing for several candidate factors (CABS_KMEANS_CAND, diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402
from workloads import CONFIGS, make_A  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dev = torch.device("cuda:0")
A = make_A(cfg, device=dev)
pipe = CabsPipeline(A, cfg.m, cfg.n, CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed))
pipe.pilot_embed()
for cf in ["1.05", "1.0003", "1.01", "1.02", "1.1", "1.2", "1.05"]:
    os.environ["CABS_KMEANS_CAND"] = cf
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.kmeans()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(cf, ["%.3f" % t for t in ts], flush=True)
