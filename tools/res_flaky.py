"""Diagnostic: repeat cabs_residual on near-factorisation inputs and report the spread against a
torch FP64 evaluation on the GPU (not a parity test: a race detector for the K > 256 plan)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402

dev = torch.device("cuda:0")
C.load()
shapes = [(40000, 640, 300), (40000, 640, 256), (40000, 640, 240), (40000, 640, 224), (40000, 640, 208), (40000, 640, 200),
          (40000, 640, 192), (40000, 640, 128), (40000, 640, 100), (100000, 640, 256), (40000, 6400, 256)]
if os.environ.get("SHAPES"):
    shapes = [tuple(int(x) for x in t.split("x")) for t in os.environ["SHAPES"].split(",")]
reps = int(os.environ.get("REPS", "12"))
for m, n, k in shapes:
    g = torch.Generator(device=dev).manual_seed(k + m)
    F = torch.randn((m, k), device=dev, generator=g) * 0.1
    G = torch.randn((n, k), device=dev, generator=g) * 0.1
    s = torch.rand(k, device=dev, generator=g) * 1.5 + 0.5
    A = ((F.double() * s.double()) @ G.double().t() + 1e-3 * torch.randn((m, n), device=dev, generator=g, dtype=torch.float64)).float()
    ref = float(((A.double() - (F.double() * s.double()) @ G.double().t()) ** 2).sum())
    plan = make_plan(m, n, k, 0, 1)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(k)
    Ft = torch.zeros((m, ld), device=dev); Ft[:, :k] = F
    Gt = torch.zeros((n, ld), device=dev); Gt[:, :k] = G
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    vals = []
    for _ in range(reps):
        C.cabs_residual(plan, A, Ft, s, Gt, k, out, ws)
        vals.append(float(out[0]))
    rel = [abs(np.sqrt(v) - np.sqrt(ref)) / np.sqrt(ref) for v in vals]
    print(f"{m}x{n} k={k}: ref {ref:.6f} distinct {len(set(vals))} max rel dev {max(rel):.2e} bad {sum(r > 1e-4 for r in rel)}/{reps}"
          f" seq {''.join('x' if r > 1e-4 else '.' for r in rel)}", flush=True)
