"""Eager vs CUDA-graph replay of one CABS step (c2) -- development probe."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402
from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402
from workloads import CHUNK, CONFIGS, Generator  # noqa: E402

cfg = CONFIGS["c2"]
dev = torch.device("cuda:0")
C.load()
plan = make_plan(cfg.m, cfg.n, max(cfg.k1, cfg.k2), 0, 1, align=CHUNK)
A = Generator(cfg, device=dev).rows(0, cfg.m)
pipe = CabsPipeline(A, cfg.m, cfg.n, CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed), 0, 1, plan=plan)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        pipe.run()
torch.cuda.synchronize()
ref = pipe.results()


def timeit(fn, n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        fn()
        e0.record(s)
        for _ in range(n):
            fn()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


t_eager = timeit(pipe.run)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    pipe.run()
torch.cuda.synchronize()
t_graph = timeit(g.replay)
got = pipe.results()
same = all(torch.equal(got[k], ref[k]) for k in ("I", "J", "Ib", "Jb", "U", "V", "lab_r", "lab_c"))
print(f"eager {t_eager:.3f} ms/step, graph replay {t_graph:.3f} ms/step, results identical: {same}, "
      f"resid {got['resid_sq']:.6e} vs {ref['resid_sq']:.6e}")
