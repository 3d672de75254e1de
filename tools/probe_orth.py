"""Leverage-variant pipeline on c2 (for an ncu launch list of its kernels)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402
from workloads import CONFIGS, make_A  # noqa: E402
dev = torch.device("cuda:0")
cfg = CONFIGS["c2"]
A = make_A(cfg, device=dev)
pipe = CabsPipeline(A, cfg.m, cfg.n, CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed, followup="leverage"))
for _ in range(3):
    pipe.run()
torch.cuda.synchronize()
print("ok", int(pipe.ro.item()))
