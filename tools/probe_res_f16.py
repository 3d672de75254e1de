"""Residual tensor-core paths at large ncomp: relative error of ||A - F diag(s) G^T||_F against
an FP64 product on the GPU, per path (FP16 split / 3xTF32 / FFMA), and the time per call.
Usage: python tools/probe_res_f16.py [m n k ...]   (set CABS_RES_F16_MAX to widen the FP16 path)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402


def run(plan, A, F, s, G, k, ws, reps=3):
    out = torch.zeros(2, dtype=torch.float64, device=A.device)
    C.cabs_residual(plan, A, F, s, G, k, out, ws)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        C.cabs_residual(plan, A, F, s, G, k, out, ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return out.cpu().tolist(), min(ts)


def main():
    a = [int(x) for x in sys.argv[1:]] or [8192, 6000, 128, 160, 192, 200, 256, 300, 320]
    m, n, ks = a[0], a[1], a[2:]
    C.load()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for k in ks:
        ld = C.cabs_padded_ld(k)
        F = torch.zeros((m, ld), device=dev); G = torch.zeros((n, ld), device=dev)
        F[:, :k] = torch.randn((m, k), device=dev, generator=g) * 0.1
        G[:, :k] = torch.randn((n, k), device=dev, generator=g) * 0.1
        s = torch.rand(k, device=dev, generator=g) * 1.5 + 0.5
        for noise in (1e-1, 1e-3):
            A = (F[:, :k].double() * s.double()) @ G[:, :k].double().T
            A = (A + noise * torch.randn((m, n), device=dev, dtype=torch.float64, generator=g)).float()
            ref = (A.double() - (F[:, :k].double() * s.double()) @ G[:, :k].double().T).pow(2).sum().sqrt().item()
            plan = make_plan(m, n, k)
            ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
            for path, env in (("f16", {"CABS_RES_F16_MAX": "384"}), ("tf32", {"CABS_RESIDUAL_TF32": "1"}),
                              ("ffma", {"CABS_RESIDUAL_FFMA": "1"})):
                old = {kk: os.environ.get(kk) for kk in ("CABS_RES_F16_MAX", "CABS_RESIDUAL_TF32", "CABS_RESIDUAL_FFMA")}
                for kk in old:
                    os.environ.pop(kk, None)
                os.environ.update(env)
                try:
                    o, t = run(plan, A, F, s, G, k, ws)
                    err = abs(o[0] ** 0.5 - ref) / ref
                    print(f"k={k} noise={noise:g} path={path:4s} ({C.cabs_residual_path(k)}) rel_err={err:.2e} "
                          f"ms={t:.3f}", flush=True)
                except Exception as e:  # noqa: BLE001
                    print(f"k={k} noise={noise:g} path={path} error {e}", flush=True)
                for kk, v in old.items():
                    os.environ.pop(kk, None)
                    if v is not None:
                        os.environ[kk] = v


if __name__ == "__main__":
    main()
