"""Debug: cabs_residual's ||A||^2 and residual vs float64 torch, per path and shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402

C.load()
dev = torch.device("cuda:0")
for (m, n, k) in [(2600, 1900, 192), (2600, 1900, 190), (2600, 1900, 128), (2600, 1900, 129), (1300, 1900, 192),
                  (2600, 1900, 250), (5000, 4000, 192)]:
    g = torch.Generator(device=dev)
    g.manual_seed(k)
    A = torch.randn((m, n), device=dev, generator=g)
    ld = C.cabs_padded_ld(k)
    F = torch.zeros((m, ld), device=dev); F[:, :k] = torch.randn((m, k), device=dev, generator=g) * 0.1
    G = torch.zeros((n, ld), device=dev); G[:, :k] = torch.randn((n, k), device=dev, generator=g) * 0.1
    plan = make_plan(m, n, k)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    C.cabs_residual(plan, A, F, None, G, k, out, ws)
    a2 = float((A.double() ** 2).sum())
    r2 = float(((A.double() - F.double() @ G.double().T) ** 2).sum())
    o = out.cpu().tolist()
    print(f"m={m} n={n} k={k}: a2 rel {abs(o[1] - a2) / a2:.2e}  r2 rel {abs(o[0] - r2) / r2:.2e}", flush=True)
