"""Simulates exact-acceleration bounds (Hamerly single lower bound; Yinyang-style group lower
bounds) for Lloyd on the real pilot embeddings of a config, FP64 in torch on the GPU: per
iteration, the fraction of points whose assignment the bounds cannot certify (they need a full
search over the centres) and the fraction that change label.  Usage: python tools/sim_bounds.py [c3]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_07395_b200 import cabs as C  # noqa: E402
from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline  # noqa: E402
from workloads import CONFIGS, make_A  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = CONFIGS[name]
dev = torch.device("cuda:0")
A = make_A(cfg, device=dev)
pipe = CabsPipeline(A, cfg.m, cfg.n, CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed))
pipe.pilot_embed()
torch.cuda.synchronize()
del A
for side, X in (("rows", pipe.P[:, :cfg.k1].double()), ("cols", pipe.Q[:, :cfg.k1].double())):
    N, k2 = X.shape[0], cfg.k2
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    cen = X[torch.randperm(N, device=dev, generator=g)[:k2]].clone()
    G = 10
    grp = torch.arange(k2, device=dev) % G
    lab = u = l = lg = None
    for it in range(cfg.iters):
        D = torch.cdist(X, cen)  # distances
        d1, j1 = D.min(1)
        Ds = D.clone()
        Ds[torch.arange(N), j1] = float("inf")
        d2 = Ds.min(1).values
        if it == 0:
            fail_h = fail_g = 1.0
        else:
            # Hamerly
            uu = u + delta[lab]
            dmax1, amax = delta.max(0)
            d2nd = delta.clone(); d2nd[amax] = 0; dmax2 = d2nd.max()
            ll = l - torch.where(lab == amax, dmax2, dmax1)
            ok1 = uu < ll
            ut = D[torch.arange(N), lab]  # tightened
            ok2 = ok1 | (ut < ll)
            fail_h = 1 - ok2.double().mean().item()
            # group bounds: lg[p, g] lower bound on distances to centres of group g (excluding own)
            dg = torch.stack([delta[grp == q].max() for q in range(G)])
            lgn = lg - dg[None, :]
            okg = (ut[:, None] < lgn).all(1)
            fail_g = 1 - okg.double().mean().item()
        changed = 0.0 if lab is None else (j1 != lab).double().mean().item()
        # exact bounds for the next iteration (as a real implementation would have after search)
        lab, u, l = j1, d1, d2
        Dg = D.clone()
        Dg[torch.arange(N), j1] = float("inf")
        lg = torch.stack([Dg[:, grp == q].min(1).values for q in range(G)], 1)
        # update
        W = torch.zeros(k2, device=dev, dtype=torch.float64).index_add_(0, lab, torch.ones(N, device=dev, dtype=torch.float64))
        S = torch.zeros_like(cen).index_add_(0, lab, X)
        new = torch.where(W[:, None] > 0, S / W.clamp_min(1)[:, None], cen)
        delta = (new - cen).norm(dim=1)
        cen = new
        print(f"{name} {side} it {it:2d}: need full search hamerly {fail_h:.4f} groups{G} {fail_g:.4f} "
              f"changed {changed:.4f} dmax {delta.max().item():.3g} dmed {delta.median().item():.3g} "
              f"med d1 {d1.median().item():.3g}", flush=True)
