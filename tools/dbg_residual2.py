import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402

C.load()
dev = torch.device("cuda:0")
m, n = 2600, 1900
for k in [int(x) for x in sys.argv[1:]] or [192]:
  for trial in range(3):
    for mode in ("rowid",):
        A = torch.ones((m, n), device=dev)
        if mode == "rowid":
            A = A * (torch.arange(m, device=dev, dtype=torch.float32)[:, None] % 97 + 1)
        ld = C.cabs_padded_ld(k)
        F = torch.zeros((m, ld), device=dev)
        G = torch.zeros((n, ld), device=dev)
        F[:, :k] = 0.01
        G[:, :k] = 0.01
        plan = make_plan(m, n, k)
        ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
        out = torch.zeros(2, dtype=torch.float64, device=dev)
        C.cabs_residual(plan, A, F, None, G, k, out, ws)
        a2 = float((A.double() ** 2).sum())
        o = out.cpu().tolist()
        print(f"k={k} trial {trial} {mode}: a2 gpu {o[1]:.1f} exact {a2:.1f} diff {o[1] - a2:.1f}", flush=True)
