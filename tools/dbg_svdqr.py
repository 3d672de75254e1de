"""SVD of zero-padded / rank-deficient inputs (QR-preconditioned quad kernel) vs LAPACK."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402

C.load()
dev = torch.device("cuda:0")
for (k, rk, pad) in [(60, 20, "rows"), (60, 20, "cols"), (60, 20, "none"), (64, 40, "none"), (100, 100, "none")]:
    g = np.random.default_rng(k + rk)
    W = (g.standard_normal((k, rk)) @ g.standard_normal((rk, k))).astype(np.float32)
    if pad == "rows":
        W[rk:, :] = 0
    if pad == "cols":
        W[:, rk:] = 0
    plan = make_plan(4 * k, 4 * k, k)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    Wt = torch.from_numpy(W).to(dev)
    sig = torch.zeros(k, dtype=torch.float64, device=dev)
    U = torch.zeros((k, k), dtype=torch.float64, device=dev)
    V = torch.zeros((k, k), dtype=torch.float64, device=dev)
    r = torch.zeros(1, dtype=torch.int32, device=dev)
    C.cabs_svd(plan, k, Wt, 1e-12, sig, U, V, r, ws)
    torch.cuda.synchronize()
    rr = int(r.item())
    s = sig.cpu().numpy(); Un = U.cpu().numpy()[:, :rr]; Vn = V.cpu().numpy()[:, :rr]
    s_ref = np.linalg.svd(W.astype(np.float64), compute_uv=False)
    rec = np.linalg.norm(W - (Un * s[:rr]) @ Vn.T) / np.linalg.norm(W)
    print(f"k={k} rank={rk} pad={pad}: r={rr} sig err {np.abs(s - s_ref).max() / s_ref[0]:.1e} rec {rec:.1e} "
          f"UtU {np.abs(Un.T @ Un - np.eye(rr)).max():.1e} VtV {np.abs(Vn.T @ Vn - np.eye(rr)).max():.1e} "
          f"status {C.cabs_device_status(ws)} sweeps {int(ws[32:36].view(torch.int32).item())}", flush=True)
    # QR timing: the two launches separately
    for env in ("", "CABS_SVD_NOQR"):
        if env:
            os.environ[env] = "1"
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            C.cabs_svd(plan, k, Wt, 1e-12, sig, U, V, r, ws)
        e1.record(); torch.cuda.synchronize()
        print(f"   {env or 'qr'}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
        if env:
            del os.environ[env]
