"""Per-phase timeline of the tensor-core Lloyd kernel (build with -DCABS_PROFILE_KTC):
runs cabs_kmeans_pair on c2/c3-shaped embeddings and prints per-iteration phase times of CTA 0."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.dist import make_plan  # noqa: E402

C.load()
dev = torch.device("cuda:0")
Na, Nb, d, k2, iters = [int(x) for x in sys.argv[1:6]] if len(sys.argv) > 5 else (100000, 50000, 100, 100, 25)
g = torch.Generator(device=dev)
g.manual_seed(1)


def emb(N):
    cen = torch.randn((64, d), device=dev, generator=g) * 3
    lab = torch.randint(0, 64, (N,), device=dev, generator=g)
    X = torch.zeros((N, C.cabs_padded_ld(d)), device=dev)
    X[:, :d] = cen[lab] + 0.05 * torch.randn((N, d), device=dev, generator=g)
    return X


Xa, Xb = emb(Na), emb(Nb)
plan = make_plan(Na, Nb, max(d, k2))
ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
ld = C.cabs_padded_ld(d)


def bufs(N):
    return (torch.zeros((k2, ld), device=dev), torch.zeros(N, dtype=torch.int32, device=dev),
            torch.zeros(k2, dtype=torch.float64, device=dev), torch.zeros(iters, dtype=torch.float64, device=dev),
            torch.zeros(iters, dtype=torch.int32, device=dev))


ba, bb = bufs(Na), bufs(Nb)
pa = C.km_problem(Xa, Na, Na, 0, d, k2, C.TAG_INIT_ROWS, *ba[:4], near_ties=ba[4])
pb = C.km_problem(Xb, Nb, Nb, 0, d, k2, C.TAG_INIT_COLS, *bb[:4], near_ties=bb[4])
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    C.cabs_kmeans_pair(plan, pa, pb, iters, C.WEIGHT_CONST, 2.0, 7, ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"kmeans_pair {Na}+{Nb} d={d} k2={k2} iters={iters}: {e0.elapsed_time(e1):.3f} ms "
          f"(path {C.cabs_kmeans_path(k2, d)}), ties {int(ba[4].sum())}/{int(bb[4].sum())}", flush=True)
allc = np.array(C.cabs_debug_counters(16 + 64 * 8 + 32 * 8)[16:])
c = allc[:64 * 8].reshape(64, 8)
tl = allc[64 * 8:].reshape(32, 8)
t0 = tl[0][0]
for t in range(32):
    if tl[t][0] == 0:
        break
    print(f"tile {t:2d}: " + " ".join(f"{(tl[t][i] - t0) / 1e3:7.2f}" for i in range(6)) + " us (load start, x_ready, mma, acc seen, cand, done)")
names = ["centres", "phaseA", "phaseB", "reduce", "barrier"]
for it in range(min(iters, 64)):
    t = c[it]
    if t[0] == 0:
        break
    nxt = c[it + 1][0] if it + 1 < 64 and c[it + 1][0] else t[5]
    print(f"it {it:2d}: " + " ".join(f"{names[i]} {(t[i + 1] - t[i]) / 1e3:6.1f}" for i in range(5)) + " us")
