"""Quick GPU probes (timings + diagnostics) for development; not part of the product path."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402


def probe_svd(k=50, reps=5, graded=False):
    dev = torch.device("cuda:0")
    plan = make_plan(1000, 1000, k)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    g = np.random.default_rng(0)
    Wn = g.standard_normal((k, k))
    if graded:  # singular values i^-1.5 plus 1e-3 noise, like W gathered from the c2 matrix
        Q1, _ = np.linalg.qr(g.standard_normal((k, k)))
        Q2, _ = np.linalg.qr(g.standard_normal((k, k)))
        Wn = (Q1 * np.arange(1, k + 1) ** -1.5) @ Q2.T + 1e-3 * Wn
    W = torch.from_numpy(Wn.astype(np.float32)).to(dev)
    sig = torch.zeros(k, dtype=torch.float64, device=dev)
    U = torch.zeros((k, k), dtype=torch.float64, device=dev)
    V = torch.zeros_like(U)
    r = torch.zeros(1, dtype=torch.int32, device=dev)
    C.cabs_svd(plan, k, W, 1e-12, sig, U, V, r, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        C.cabs_svd(plan, k, W, 1e-12, sig, U, V, r, ws)
    e1.record()
    torch.cuda.synchronize()
    sweeps = int(ws[32:36].view(torch.int32).item())
    Wd = W.double().cpu().numpy()
    sv = np.linalg.svd(Wd, compute_uv=False)
    Uh, Vh, sh = U.cpu().numpy(), V.cpu().numpy(), sig.cpu().numpy()
    rec = np.linalg.norm(Uh * sh @ Vh.T - Wd) / np.linalg.norm(Wd)
    Ul, sl, Vlt = np.linalg.svd(Wd)
    sgn = np.sign(np.sum(Ul * Uh, axis=0)); sgn[sgn == 0] = 1
    udiff = np.abs(Uh * sgn - Ul).max()
    orth = max(np.abs(Uh.T @ Uh - np.eye(k)).max(), np.abs(Vh.T @ Vh - np.eye(k)).max())
    print(f"svd k={k}{' graded' if graded else ''}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us/call, sweeps={sweeps}, "
          f"r={int(r.item())}, sigma rel err {np.abs(sh - sv).max() / sv[0]:.1e}, recon {rec:.1e}, orth {orth:.1e}, "
          f"U vs LAPACK {udiff:.1e}")


def probe_residual(m=20000, n=10000, k=50, reps=5):
    dev = torch.device("cuda:0")
    plan = make_plan(m, n, k)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    A = torch.randn(m, n, device=dev)
    ld = C.cabs_padded_ld(k)
    F = torch.zeros(m, ld, device=dev); F[:, :k] = torch.randn(m, k, device=dev) * 0.1
    G = torch.zeros(n, ld, device=dev); G[:, :k] = torch.randn(n, k, device=dev) * 0.1
    s = torch.rand(k, device=dev) + 0.5
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    C.cabs_residual(plan, A, F, s, G, k, out, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        C.cabs_residual(plan, A, F, s, G, k, out, ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ref_r = ((A.double() - (F[:, :k].double() * s.double()) @ G[:, :k].double().T) ** 2).sum().item()
    print(f"residual {m}x{n} k={k}: {ms * 1e3:.1f} us, {4 * m * n / ms / 1e6:.0f} GB/s, "
          f"rel diff {abs(out[0].item() - ref_r) / ref_r:.2e}, a2 rel {abs(out[1].item() - (A.double()**2).sum().item()) / out[1].item():.1e}")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("svd", "all"):
        for k in (2, 3, 16, 20, 33, 50, 64, 100, 200):
            probe_svd(k)
        for k in (20, 50, 64):
            probe_svd(k, graded=True)
    if what in ("residual", "all"):
        for (m, n, k) in ((20000, 10000, 50), (2000, 1500, 20), (20000, 10000, 64), (4097, 3001, 33)):
            probe_residual(m, n, k)


def probe_kmeans(N=20000, d=50, k2=50, iters=20, reps=3):
    dev = torch.device("cuda:0")
    plan = make_plan(N, N, max(d, k2))
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(d)
    X = torch.zeros(N, ld, device=dev); X[:, :d] = torch.randn(N, d, device=dev)
    cen = torch.zeros(k2, ld, device=dev); lab = torch.zeros(N, dtype=torch.int32, device=dev)
    cw = torch.zeros(k2, dtype=torch.float64, device=dev); obj = torch.zeros(iters, dtype=torch.float64, device=dev)
    C.cabs_kmeans(plan, X, N, N, 0, d, k2, iters, 0, 2.0, 0, 3, cen, lab, cw, obj, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        C.cabs_kmeans(plan, X, N, N, 0, d, k2, iters, 0, 2.0, 0, 3, cen, lab, cw, obj, ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"kmeans N={N} d={d} k2={k2} iters={iters}: {ms * 1e3:.1f} us ({ms * 1e3 / iters:.1f} us/iter)")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] in ("kmeans", "all2"):
    for cfg in ((20000, 50, 50), (10000, 50, 50), (100000, 100, 100), (2000, 20, 20)):
        probe_kmeans(*cfg)


def probe_svd_prof(k=50):
    """Needs libcabs built with -DCABS_PROFILE_SVD: per-phase cycles of warp 0 summed over rounds."""
    dev = torch.device("cuda:0")
    plan = make_plan(1000, 1000, k)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    g = np.random.default_rng(0)
    W = torch.from_numpy(g.standard_normal((k, k)).astype(np.float32)).to(dev)
    sig = torch.zeros(k, dtype=torch.float64, device=dev)
    r = torch.zeros(1, dtype=torch.int32, device=dev)
    C.cabs_svd(plan, k, W, 1e-12, sig, None, None, r, ws)
    torch.cuda.synchronize()
    sweeps = int(ws[32:36].view(torch.int32).item())
    prof = ws[64:128].view(torch.int64).tolist()
    rounds = sweeps * (k + (k % 2))
    names = ["dots", "butterfly", "angle", "rotate+params", "publish", "barrier", "loads", "loop/other"]
    print(f"k={k} sweeps={sweeps} rounds~{rounds}: " + ", ".join(f"{n} {p / max(rounds, 1):.0f} cyc" for n, p in zip(names, prof)))


def probe_svd_quad_prof(k=50):
    """Needs -DCABS_PROFILE_SVD: per-CTA wait / round-loop / total cycles."""
    dev = torch.device("cuda:0")
    plan = make_plan(1000, 1000, k)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    g = np.random.default_rng(0)
    W = torch.from_numpy(g.standard_normal((k, k)).astype(np.float32)).to(dev)
    sig = torch.zeros(k, dtype=torch.float64, device=dev)
    r = torch.zeros(1, dtype=torch.int32, device=dev)
    C.cabs_svd(plan, k, W, 1e-12, sig, None, None, r, ws)
    torch.cuda.synchronize()
    sweeps = int(ws[32:36].view(torch.int32).item())
    p = ws[64:144].view(torch.int64).tolist()
    print(f"  CTA0: start->loop {p[6]}, loop->epilogue {p[7]}, sigma {p[8]}, write {p[9]} cycles")
    rounds = sweeps * ((k + 3) & ~3)
    print(f"k={k} sweeps={sweeps}: CTA0 wait {p[0]} rounds {p[1]} ({p[1] / rounds:.0f}/round) total {p[2]}; "
          f"CTA1 wait {p[3]} rounds {p[4]} ({p[4] / rounds:.0f}/round) total {p[5]}")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "svdqprof":
    for kk in [int(x) for x in sys.argv[2:]] or [50, 20]:
        probe_svd_quad_prof(kk)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "svdprof":
    for k in (20, 50):
        probe_svd_prof(k)


def probe_lloyd_prof(N=20000, d=50, k2=50, iters=20):
    """Needs libcabs built with -DCABS_PROFILE_LLOYD: per-phase cycles of CTA 0 per iteration."""
    dev = torch.device("cuda:0")
    plan = make_plan(N, N, max(d, k2))
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(d)
    X = torch.zeros(N, ld, device=dev); X[:, :d] = torch.randn(N, d, device=dev)
    cen = torch.zeros(k2, ld, device=dev); lab = torch.zeros(N, dtype=torch.int32, device=dev)
    cw = torch.zeros(k2, dtype=torch.float64, device=dev); obj = torch.zeros(iters, dtype=torch.float64, device=dev)
    C.cabs_kmeans(plan, X, N, N, 0, d, k2, iters, 0, 2.0, 0, 3, cen, lab, cw, obj, ws)
    torch.cuda.synchronize()
    prof = ws[64:144].view(torch.int64).tolist()
    names = ["centres+zero", "dist+argmin", "bucket", "obj-publish", "barrier", "cluster.sync1", "dsmem-reduce+red",
             "fence", "cluster.sync2"]
    print(f"lloyd N={N} d={d} k2={k2}: " + ", ".join(f"{n} {p / iters:.0f} cyc" for n, p in zip(names, prof)))


def probe_lloyd_pair(Na=20000, Nb=10000, d=50, k2=50, iters=20, prof=False):
    """cabs_kmeans_pair timing (and, with -DCABS_PROFILE_LLOYD, per-phase cycles of the last CTA)."""
    dev = torch.device("cuda:0")
    plan = make_plan(Na, Nb, max(d, k2))
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(d)
    bufs = []
    probs = []
    for N, tag in ((Na, 3), (Nb, 4)):
        X = torch.zeros(N, ld, device=dev); X[:, :d] = torch.randn(N, d, device=dev)
        b = (X, torch.zeros(k2, ld, device=dev), torch.zeros(N, dtype=torch.int32, device=dev),
             torch.zeros(k2, dtype=torch.float64, device=dev), torch.zeros(iters, dtype=torch.float64, device=dev))
        bufs.append(b)
        probs.append(C.km_problem(b[0], N, N, 0, d, k2, tag, b[1], b[2], b[3], b[4]))
    C.cabs_kmeans_pair(plan, probs[0], probs[1], iters, 0, 2.0, 0, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        C.cabs_kmeans_pair(plan, probs[0], probs[1], iters, 0, 2.0, 0, ws)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3 * 1e3
    line = f"kmeans_pair Na={Na} Nb={Nb} d={d} k2={k2} iters={iters}: {t:.1f} us ({t / iters:.1f} us/iter)"
    if prof:
        p = ws[64:144].view(torch.int64).tolist()
        names = ["centres+zero", "dist+merge", "accum", "grid barrier", "-", "cluster.sync", "dsmem-reduce+red"]
        line += "\n  " + ", ".join(f"{n} {v / iters:.0f}" for n, v in zip(names, p) if n != "-")
    print(line)


def lloyd_timeline(G=148):
    """Per-CTA phase stamps of iteration 10 (-DCABS_PROFILE_LLOYD): duration statistics over
    the CTAs, and where the iteration's critical path goes (relative to the first CTA's start)."""
    t = np.array(C.cabs_debug_counters(16 + 320 * 16), dtype=np.int64)[16:].reshape(320, 16)
    t = t[(t[:, 0] > 0)]
    names = ["top", "mbar", "centres", "dist", "acc", "csync", "reduce", "prebar", "passbar"]
    t = t[:, :len(names)].astype(np.float64)
    t0 = t[:, 0].min()
    print(f"  timeline of {t.shape[0]} CTAs (ns; start = first CTA at iteration top)")
    for i in range(1, len(names)):
        dur = t[:, i] - t[:, i - 1]
        print(f"    {names[i]:8s} dur min {dur.min():7.0f} med {np.median(dur):7.0f} max {dur.max():7.0f}"
              f" | reached at min {t[:, i].min() - t0:7.0f} max {t[:, i].max() - t0:7.0f}")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "lloydpair":
    probe_lloyd_pair(prof=len(sys.argv) > 2)
    if len(sys.argv) > 2:
        lloyd_timeline()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "lloydprof":
    for cfg in ((20000, 50, 50), (10000, 50, 50), (100000, 100, 100)):
        probe_lloyd_prof(*cfg)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "resprof":
    probe_residual(20000, 10000, 50, reps=1)
    c = C.cabs_debug_counters(16)
    names = {0: "prod wait f_empty", 1: "prod wait a_empty", 2: "prod wait g_empty", 3: "prod total",
             4: "mma wait f_full", 5: "mma wait g_split", 6: "mma wait acc_empty", 7: "mma total",
             8: "split wait g_full", 9: "split total", 10: "epi wait a_full", 11: "epi wait acc_full", 12: "epi total"}
    for i, nm in names.items():
        print(f"{nm:22s} {c[i]:12d} cycles")
