"""GPU parity of the NEXT-4 baselines: BR-CUR (Algorithm 1) and
Sketch-CUR (P:115, P:312 (a)) through cabs_br_cur against the oracle's br_cur / sketch_cur, and
the validation rank sweep through cabs_holdout_errors against the oracle's
holdout_errors / validate_rank."""
import math

import numpy as np
import pytest
import torch

from oracle import cabs as O
from oracle import rng
from tests.helpers import rel_fro

pytestmark = pytest.mark.gpu

C = pytest.importorskip("paper_1607_07395_b200.cabs")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    C.load()
    return torch.device("cuda:0")


def _A(m, n, r, noise, seed):
    g = np.random.default_rng(seed)
    A = (g.standard_normal((m, r)) / np.arange(1, r + 1)) @ g.standard_normal((r, n)) + noise * g.standard_normal((m, n))
    return A.astype(np.float32)


@pytest.mark.parametrize("m,n,k1,k2,rank,noise", [(900, 700, 20, 60, 30, 0.01), (2000, 1500, 12, 12, 12, 0.0),
                                                  (1500, 3000, 50, 150, 200, 0.05), (600, 800, 40, 100, 40, 0.0)])
def test_br_cur_matches_oracle(dev, m, n, k1, k2, rank, noise):
    from paper_1607_07395_b200.dist import make_plan
    A = _A(m, n, rank, noise, m + k1)
    g = np.random.default_rng(k2)
    Ibr, Ibc = np.sort(g.choice(m, k1, replace=False)), np.sort(g.choice(n, k1, replace=False))
    Itr, Itc = np.sort(g.choice(m, k2, replace=False)), np.sort(g.choice(n, k2, replace=False))
    if k2 == k1:  # coincident base / target sampling: the pseudo-skeleton (section 2.2 item 2)
        Itr, Itc = Ibr, Ibc
    plan = make_plan(m, n, k2)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    At = torch.from_numpy(A).to(dev)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    ld = C.cabs_padded_ld(k1)
    F, G = torch.zeros((m, ld), device=dev), torch.zeros((n, ld), device=dev)
    Um = torch.zeros((k1, k1), dtype=torch.float64, device=dev)
    C.cabs_br_cur(plan, At, k1, t(Ibr), t(Ibc), k2, t(Itr), t(Itc), F, G, ws, Umid=Um)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    C.cabs_residual(plan, At, F, None, G, k1, out, ws)
    torch.cuda.synchronize()
    ref = O.br_cur(A, Ibr, Ibc, Itr, Itc)
    assert np.array_equal(G.cpu().numpy()[:, :k1], ref.R.T.astype(np.float32))  # R^T: exact copies
    Fr = ref.C @ ref.U
    assert rel_fro(F.cpu().numpy()[:, :k1], Fr) < 1e-4
    r2, a2 = O.residual(A, Fr, ref.R.T)
    assert abs(out[1].item() - a2) <= 1e-6 * a2
    if noise == 0.0 and k1 >= rank:
        # exact recovery (both sides): the oracle to FP64 rounding, the GPU to the FP32 floor of
        # the reconstruction (F = C U* in FP32, the fused residual's products)
        assert r2 <= 1e-9 * a2 and out[0].item() <= 1e-8 * a2  # A is the FP32 rounding of a rank-k matrix
    else:
        assert abs(math.sqrt(max(out[0].item(), 0)) - math.sqrt(r2)) <= 1e-4 * math.sqrt(r2) + 1e-6 * math.sqrt(a2)


def test_sketch_cur_matches_oracle(dev):
    from paper_1607_07395_b200.pipeline import SketchCurRun
    from workloads import CONFIGS, make_A, scaled
    cfg = scaled(CONFIGS["c1"], 2000, 1500, k1=20, seed=3)
    A_t = make_A(cfg, device=dev)
    A = A_t.cpu().numpy()
    run = SketchCurRun(A_t, cfg.m, cfg.n, 20, mult=3, seed=3)
    run.run()
    torch.cuda.synchronize()
    I, J = rng.floyd(cfg.m, 20, 3, rng.TAG_PILOT_ROWS), rng.floyd(cfg.n, 20, 3, rng.TAG_PILOT_COLS)
    ref, Itr, Itc = O.sketch_cur(A, I, J, 3, seed=3)
    assert np.array_equal(run.Ibr.cpu().numpy(), I) and np.array_equal(run.Itr.cpu().numpy(), Itr)
    assert np.array_equal(run.Itc.cpu().numpy(), Itc)
    r2, a2 = O.residual(A, ref.C @ ref.U, ref.R.T)
    rg = math.sqrt(max(run.out[0].item(), 0))
    assert abs(rg - math.sqrt(r2)) <= 1e-4 * math.sqrt(r2) + 1e-6 * math.sqrt(a2)
    assert rel_fro(run.Umid.cpu().numpy(), ref.U) < 1e-4


@pytest.mark.parametrize("name,m,n,k,h", [("c1", 2000, 1500, 20, 20), ("c2", 6000, 3000, 50, 50),
                                          ("c3", 5000, 2500, 100, 100)])
def test_rank_sweep_matches_oracle(dev, name, m, n, k, h):
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline, rank_sweep
    from workloads import CONFIGS, make_A, scaled
    cfg = scaled(CONFIGS[name], m, n, k1=k, k2=k, iters=4, seed=1)
    A_t = make_A(cfg, device=dev)
    A = A_t.cpu().numpy()
    pipe = CabsPipeline(A_t, m, n, CabsConfig(k, k, 4, seed=1))
    pipe.run()
    e, rank, Hr, Hc = rank_sweep(pipe, h)
    r = int(pipe.r2.item())
    U = pipe.U.cpu().numpy()[:, :r].astype(np.float64)
    V = pipe.V.cpu().numpy()[:, :r].astype(np.float64)
    s = pipe.s2.cpu().numpy()[:r].astype(np.float64)
    Hr_o = O.holdout_indices(m, h, 1, rng.TAG_HOLDOUT_ROWS, pipe.Ib.cpu().numpy())
    Hc_o = O.holdout_indices(n, h, 1, rng.TAG_HOLDOUT_COLS, pipe.Jb.cpu().numpy())
    assert np.array_equal(Hr.numpy(), Hr_o) and np.array_equal(Hc.numpy(), Hc_o)
    ref = O.holdout_errors(A, U, s, V, Hr_o, Hc_o)   # the oracle's sweep on the GPU's factors
    assert e.shape[0] == r + 1
    assert np.abs(e.numpy() - ref).max() <= 1e-6 * ref[0]
    want = O.validate_rank(ref)
    assert rank == want or abs(ref[rank] - ref[want]) <= 1e-6 * ref[0]
