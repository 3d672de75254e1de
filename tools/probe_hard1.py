import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402
dev = torch.device("cuda:0")
N, d, k2 = 20000, 50, 50
plan = make_plan(N, N, 64)
ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
X = torch.zeros((N, 64), device=dev)
X[:, :d] = torch.randn(N, d, device=dev)
reps = torch.zeros(k2, dtype=torch.int64, device=dev)
for _ in range(3):
    C.cabs_hard_select(plan, X, N, N, 0, d, k2, reps, ws)
torch.cuda.synchronize()
print("ok")
