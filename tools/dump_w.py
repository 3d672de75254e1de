"""Dumps the two k x k SVD inputs of a full-size config (W = A(I, J) of the pilot, W_bar =
A(I_bar, J_bar) of the sketch) and the sweep counts the library's SVD needed, for offline
convergence studies.  Usage: python tools/dump_w.py [c3] -> gpurun_out/w_<cfg>.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402
from workloads import CONFIGS, make_A  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = CONFIGS[name]
dev = torch.device("cuda:0")
A = make_A(cfg, device=dev)
pipe = CabsPipeline(A, cfg.m, cfg.n, CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed))
pipe.pilot_embed()
torch.cuda.synchronize()
sw1 = int(pipe.ws[32:36].view(torch.int32).item())
pipe.kmeans(); pipe.select(); pipe.sketch()
torch.cuda.synchronize()
sw2 = int(pipe.ws[32:36].view(torch.int32).item())
k1, k2 = cfg.k1, cfg.k2
W = pipe.W[:, :k1].cpu().numpy()
Ib, Jb = pipe.Ib.cpu(), pipe.Jb.cpu()
Wb = A[Ib.to(dev)][:, Jb.to(dev)].cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/w_{name}.npz", W=W, Wb=Wb, sweeps=np.array([sw1, sw2]))
print(name, "sweeps", sw1, sw2, "sigma1", pipe.sigma1[:5].tolist(), "...", pipe.sigma1[-3:].tolist())
