"""Times cabs_residual alone on a c3-shaped problem (m x n FP32 A in HBM, ncomp factors):
CUDA events around each call, L2 flushed in between.  Usage: python tools/time_residual.py [m n k ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]] or [100000, 50000, 100]
    m, n = a[0], a[1]
    ks = a[2:] or [100]
    C.load()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    A = torch.randn((m, n), device=dev, generator=g)
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    for k in ks:
        ld = C.cabs_padded_ld(k)
        F = torch.randn((m, ld), device=dev, generator=g) * 0.1
        G = torch.randn((n, ld), device=dev, generator=g) * 0.1
        F[:, k:] = 0
        G[:, k:] = 0
        plan = make_plan(m, n, k)
        ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
        out = torch.zeros(2, dtype=torch.float64, device=dev)
        for _ in range(3):
            C.cabs_residual(plan, A, F, None, G, k, out, ws)
        ts = []
        for _ in range(5):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            C.cabs_residual(plan, A, F, None, G, k, out, ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = min(ts)
        if os.environ.get("RESPROF"):
            c = C.cabs_debug_counters(16)
            names = {1: "A prod wait a_empty", 2: "G prod wait g_empty", 3: "A prod total", 4: "mma wait f_ready",
                     5: "mma wait g_full", 6: "mma wait acc_empty", 7: "mma total", 10: "epi wait a_full",
                     11: "epi wait acc_full", 12: "epi total"}
            print("  " + ", ".join(f"{nm}={c[i]}" for i, nm in names.items()))
        gb = 4.0 * (m * n + m * k + n * k) / 1e9
        print(f"m={m} n={n} k={k} path={C.cabs_residual_path(k)} ms={t:.3f} (all {['%.3f' % x for x in ts]}) "
              f"GB/s={gb / t * 1e3:.0f} frac={gb / t * 1e3 / 6554.9:.3f}")


if __name__ == "__main__":
    main()
