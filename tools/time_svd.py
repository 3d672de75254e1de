"""Times cabs_svd (S4) for several k and checks it against LAPACK: sigma error / sigma_1,
||U^T U - I||, ||V^T V - I||, ||W - U S V^T|| / ||W||, and the sweep count (ws[8]).
Usage: python tools/time_svd.py [k ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402

C.load()
dev = torch.device("cuda:0")
for k in [int(x) for x in sys.argv[1:]] or [50, 64, 100, 128, 200, 300]:
    g = np.random.default_rng(k)
    W = (g.standard_normal((k, k)) @ np.diag(np.logspace(0, -6, k)) @ g.standard_normal((k, k))).astype(np.float32)
    plan = make_plan(4 * k, 4 * k, k)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(k)
    Wt = torch.zeros((k, ld), device=dev); Wt[:, :k] = torch.from_numpy(W).to(dev)
    sig = torch.zeros(k, dtype=torch.float64, device=dev)
    U = torch.zeros((k, k), dtype=torch.float64, device=dev)
    V = torch.zeros((k, k), dtype=torch.float64, device=dev)
    r = torch.zeros(1, dtype=torch.int32, device=dev)
    for _ in range(2):
        C.cabs_svd(plan, k, Wt, 1e-12, sig, U, V, r, ws)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        C.cabs_svd(plan, k, Wt, 1e-12, sig, U, V, r, ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    sweeps = int(ws[32:36].view(torch.int32).item())
    s_ref = np.linalg.svd(W.astype(np.float64), compute_uv=False)
    s = sig.cpu().numpy(); Un = U.cpu().numpy(); Vn = V.cpu().numpy(); rr = int(r.item())
    Ur, Vr = Un[:, :rr], Vn[:, :rr]
    rec = np.linalg.norm(W - (Ur * s[:rr]) @ Vr.T) / np.linalg.norm(W)
    print(f"k={k:3d} {min(ts):8.3f} ms  sweeps={sweeps:2d} r={rr}  sigma err {np.max(np.abs(s - s_ref)) / s_ref[0]:.1e}  "
          f"UtU {np.abs(Ur.T @ Ur - np.eye(rr)).max():.1e}  VtV {np.abs(Vr.T @ Vr - np.eye(rr)).max():.1e}  "
          f"rec {rec:.1e}  status {C.cabs_device_status(ws)}", flush=True)
    if os.environ.get("SVDPROF"):
        pc = ws[128:160].view(torch.int64).cpu().tolist()
        print("   cycles: within-block %d, cross %d, seat changes %d, convergence %d" % tuple(pc), flush=True)
