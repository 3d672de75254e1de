"""Time cabs_hard_select (P:312 variant (f)) on c2-sized embeddings and the hard-threshold pipeline step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402

dev = torch.device("cuda:0")
for N, d, k2 in ((20000, 50, 50), (10000, 50, 50), (400000, 200, 200)):
    plan = make_plan(N, N, max(d, k2))
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    X = torch.zeros((N, C.cabs_padded_ld(d)), device=dev)
    X[:, :d] = torch.randn(N, d, device=dev)
    reps = torch.zeros(k2, dtype=torch.int64, device=dev)
    for _ in range(3):
        C.cabs_hard_select(plan, X, N, N, 0, d, k2, reps, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        C.cabs_hard_select(plan, X, N, N, 0, d, k2, reps, ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"hard_select N={N} d={d} k2={k2}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")

from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402
from workloads import CONFIGS, make_A  # noqa: E402
cfg = CONFIGS["c2"]
A = make_A(cfg, device=dev)
for fu in ("kmeans", "hard"):
    pipe = CabsPipeline(A, cfg.m, cfg.n, CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed, followup=fu))
    for _ in range(3):
        pipe.run(timed=True)
    pipe.step_ms()
    pipe.run(timed=True)
    ms = pipe.step_ms()
    g = pipe.results()
    print(fu, {k: round(v, 4) for k, v in ms.items()}, "total", round(sum(ms.values()), 4),
          "relerr", (g["resid_sq"] / g["a_sq"]) ** 0.5)
