"""Per-phase timeline and candidate counts of the tensor-core Lloyd kernel on the REAL c3
embeddings (pilot sketch of the c3 matrix), build with -DCABS_PROFILE_KTC.
Usage: python tools/prof_ktc_c3.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402
from workloads import CONFIGS, make_A  # noqa: E402

C.load()
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = CONFIGS[name]
dev = torch.device("cuda:0")
A = make_A(cfg, device=dev)
pipe = CabsPipeline(A, cfg.m, cfg.n, CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed))
pipe.pilot_embed()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pipe.kmeans()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} kmeans_pair: {e0.elapsed_time(e1):.3f} ms (path {C.cabs_kmeans_path(cfg.k2, cfg.k1)}) "
          f"ties {int(pipe.tie_r.sum())}/{int(pipe.tie_c.sum())}", flush=True)
P = pipe.P[:, :cfg.k1].float()
Q = pipe.Q[:, :cfg.k1].float()
for nm, X, cen in (("rows", P, pipe.cen_r[:, :cfg.k1]), ("cols", Q, pipe.cen_c[:, :cfg.k1])):
    x2 = (X * X).sum(1)
    d = torch.cdist(X[:20000], cen) ** 2
    dm = d.min(1).values
    print(f"{nm}: median ||x||^2 {x2.median():.4g}, median nearest d^2 {dm.median():.4g}, "
          f"ratio {float((x2[:20000] / dm.clamp_min(1e-30)).median()):.4g}")
allc = np.array(C.cabs_debug_counters(16 + 64 * 8 + 32 * 8 + 64 * 2)[16:])
c = allc[:64 * 8].reshape(64, 8)
tl = allc[64 * 8:64 * 8 + 32 * 8].reshape(32, 8)
cand = allc[64 * 8 + 32 * 8:].reshape(64, 2)
t0 = tl[0][0]
for t in range(32):
    if tl[t][0] == 0:
        break
    print(f"tile {t:2d}: " + " ".join(f"{(tl[t][i] - t0) / 1e3:7.2f}" for i in range(6)) +
          " us (load start, x_ready, mma, acc seen, cand, done)")
names = ["centres", "phaseA", "phaseB", "reduce", "barrier"]
for it in range(min(cfg.iters, 64)):
    t = c[it]
    if t[0] == 0:
        break
    print(f"it {it:2d}: " + " ".join(f"{names[i]} {(t[i + 1] - t[i]) / 1e3:6.1f}" for i in range(5)) + " us"
          + (f"  cand/pt {cand[it][1] / max(cand[it][0], 1):.2f}" if cand[it][0] else ""))
