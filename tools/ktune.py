"""c3 k-means pair timing over (Dn refresh period, full-iteration divisor) -- diagnostics."""
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
for dp, fd in [p.split(":") for p in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["4:16", "8:16", "4:8", "8:8"])]:
    os.environ["CABS_KM_DPERIOD"] = dp
    os.environ["CABS_KM_FULLDIV"] = fd
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.kmeans()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(dp, fd, ["%.3f" % t for t in ts], flush=True)
