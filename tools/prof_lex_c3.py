"""Per-phase timeline of the pruned Lloyd kernel on the REAL embeddings of a config (build with
-DCABS_PROFILE_LEX), plus the timing of the other k-means paths for comparison.
Usage: python tools/prof_lex_c3.py [config]"""
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
res = {}
for cf in os.environ.get("CANDS", "1.05").split():
    os.environ["CABS_KMEANS_CAND"] = cf
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.kmeans()
        e1.record()
        torch.cuda.synchronize()
    print(f"cand factor {cf}: {e0.elapsed_time(e1):.3f} ms", flush=True)
    del os.environ["CABS_KMEANS_CAND"]
for env in ("", "CABS_KMEANS_TC", "CABS_KMEANS_FFMA"):
    if env:
        os.environ[env] = "1"
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.kmeans()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
    print(f"{name} kmeans_pair path {C.cabs_kmeans_path(cfg.k2, cfg.k1)}: {t:.3f} ms, ties "
          f"{int(pipe.tie_r.sum())}/{int(pipe.tie_c.sum())}", flush=True)
    res[env] = (pipe.lab_r.cpu().numpy().copy(), pipe.lab_c.cpu().numpy().copy(), pipe.cen_r.cpu().numpy().copy(),
                pipe.cen_c.cpu().numpy().copy())
    if env == "":
        raw = np.array(C.cabs_debug_counters(16 + 64 * 16 + 64)[16:])
        allc = raw[:1024].reshape(64, 16)
        qn = raw[1024:]
    if env:
        del os.environ[env]
for env in ("CABS_KMEANS_TC", "CABS_KMEANS_FFMA"):
    same = all(np.array_equal(a, b) for a, b in zip(res[""], res[env]))
    print(f"prune vs {env}: labels and centres identical: {same}")
N = cfg.m + cfg.n
for it in range(min(cfg.iters, 64)):
    t = allc[it]
    if t[0] == 0:
        break
    seq = [("Sl", 8), ("obj", 9), ("centres", 1), ("D", 2), ("bound", 6), ("search", 3), ("reduce", 4), ("barrier", 5)]
    prev, out = t[0], []
    for nm, i in seq:
        if t[i]:
            out.append(f"{nm} {(t[i] - prev) / 1e3:6.1f}")
            prev = t[i]
    print(f"it {it:2d}: " + " ".join(out) + f" us  queued {qn[it] / 3 / N:.3f}  union cand/queued pt {t[7] / max(qn[it], 1):.2f}")
