"""GPU parity of the implicit RBF source (c5, BASELINE.json configs[4]) and of the sampled
residual, through the C ABI, against the FP64 oracle (oracle.cabs.RbfSource,
oracle.cabs.residual_sampled, oracle.rng.residual_pairs).

* pair positions: bit-exact (integer Philox + Lemire on both sides);
* generated entries: FP32 direct differences + ex2.approx vs FP64: |err| <= 2e-6 (entries in (0, 1]);
* sampled residual: same pairs on both sides; r within 1e-4 r + 1e-6 a, a^2 within 1e-6;
* end to end at reduced c5 sizes with first-divergence parity (tests/parity.py).
"""
import math

import numpy as np
import pytest
import torch

from oracle import cabs as O
from oracle import rng

pytestmark = pytest.mark.gpu

C = pytest.importorskip("paper_1607_07395_b200.cabs")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    C.load()
    return torch.device("cuda:0")


def _rbf(m, n, d, seed, dev):
    from workloads import CONFIGS, make_rbf, scaled
    if d == 16:
        x, y, sigma = make_rbf(scaled(CONFIGS["c5"], m, n, seed=seed))
    else:
        g = np.random.default_rng(seed)
        x = torch.from_numpy(g.standard_normal((m, d)).astype(np.float32))
        y = torch.from_numpy(g.standard_normal((n, d)).astype(np.float32))
        sigma = 1.3
    return C.RbfSource(x.to(dev), y.to(dev), sigma), O.RbfSource(x.numpy(), y.numpy(), sigma)


@pytest.mark.parametrize("m,n,T,t0", [(2000000, 1000000, 1 << 20, 0), ((1 << 31) + 1, (1 << 31) + 1, 100000, 0),
                                      (7, 5, 50000, 12345), (1, 1, 10, 0), ((1 << 32), 3, 4096, 1 << 33)])
def test_residual_pairs_bit_exact(dev, m, n, T, t0):
    i = torch.zeros(T, dtype=torch.int64, device=dev)
    j = torch.zeros(T, dtype=torch.int64, device=dev)
    C.cabs_residual_pairs(11, t0, T, m, n, i, j)
    ri, rj = rng.residual_pairs(11, T, m, n, t0=t0)
    assert np.array_equal(i.cpu().numpy(), ri) and np.array_equal(j.cpu().numpy(), rj)


@pytest.mark.parametrize("m,n,k,d", [(5000, 4000, 60, 16), (3001, 1999, 33, 5), (700, 900, 300, 16)])
def test_rbf_gathers_match_oracle(dev, m, n, k, d):
    from paper_1607_07395_b200.dist import make_plan
    src, osrc = _rbf(m, n, d, 7, dev)
    plan = make_plan(m, n, k)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(k)
    I, J = torch.zeros(k, dtype=torch.int64, device=dev), torch.zeros(k, dtype=torch.int64, device=dev)
    Cm, R, W = torch.zeros((m, ld), device=dev), torch.zeros((k, (n + 3) // 4 * 4), device=dev), torch.zeros((k, ld), device=dev)
    C.cabs_pilot(plan, src, k, 5, I, J, Cm, R, W, ws)
    Ih, Jh = I.cpu().numpy(), J.cpu().numpy()
    assert np.array_equal(Ih, rng.floyd(m, k, 5, rng.TAG_PILOT_ROWS))
    assert np.array_equal(Jh, rng.floyd(n, k, 5, rng.TAG_PILOT_COLS))
    Co, Ro, Wo = O.gather(osrc, Ih, Jh)
    assert np.abs(Cm.cpu().numpy()[:, :k] - Co).max() < 2e-6
    assert np.abs(R.cpu().numpy()[:, :n] - Ro).max() < 2e-6
    assert np.abs(W.cpu().numpy()[:, :k] - Wo).max() < 2e-6
    # generate-on-access is a function of (i, j) only: W from cabs_pilot_embed's direct path, R[:, J]
    # and C[I, :] are the same bits
    W2 = torch.zeros_like(W)
    P, Q = torch.zeros((m, ld), device=dev), torch.zeros((n, ld), device=dev)
    s, r = torch.zeros(k, device=dev), torch.zeros(1, dtype=torch.int32, device=dev)
    C.cabs_pilot_embed(plan, src, k, 5, I, J, Cm, R, W2, C.STABILIZED, 1e-12, P, Q, s, r, ws)
    torch.cuda.synchronize()
    assert torch.equal(W2[:, :k], W[:, :k])
    assert torch.equal(R[:, J], W[:, :k]) and torch.equal(Cm[I, :k], W[:, :k])


@pytest.mark.parametrize("kind", ["dense", "rbf"])
@pytest.mark.parametrize("ncomp", [1, 37, 60, 300])
def test_residual_sampled_matches_oracle(dev, kind, ncomp):
    from paper_1607_07395_b200.dist import make_plan
    m, n, T, seed = 3000, 2000, 1 << 20, 9
    g = np.random.default_rng(ncomp)
    F = g.standard_normal((m, ncomp)).astype(np.float32) * 0.1
    G = g.standard_normal((n, ncomp)).astype(np.float32) * 0.1
    sv = g.uniform(0.5, 2.0, ncomp).astype(np.float32)
    if kind == "dense":
        A = (F @ G.T * sv[0] + 0.05 * g.standard_normal((m, n))).astype(np.float32)
        src, osrc = torch.from_numpy(A).to(dev), A
    else:
        src, osrc = _rbf(m, n, 16, 3, dev)
    plan = make_plan(m, n, max(ncomp, 1))
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(ncomp)
    Ft, Gt = torch.zeros((m, ld), device=dev), torch.zeros((n, ld), device=dev)
    Ft[:, :ncomp], Gt[:, :ncomp] = torch.from_numpy(F).to(dev), torch.from_numpy(G).to(dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    C.cabs_residual(plan, src, Ft, torch.from_numpy(sv).to(dev), Gt, ncomp, out, ws, n_samples=T, seed=seed)
    i, j = rng.residual_pairs(seed, T, m, n)
    r2, a2 = O.residual_sampled(osrc, F, G, i, j, sv)
    o = out.cpu().numpy()
    assert abs(o[1] - a2) <= 1e-6 * a2
    assert abs(math.sqrt(o[0]) - math.sqrt(r2)) <= 1e-4 * math.sqrt(r2) + 1e-6 * math.sqrt(a2)
    # deterministic: a second call gives the same bits
    out2 = torch.zeros_like(out)
    C.cabs_residual(plan, src, Ft, torch.from_numpy(sv).to(dev), Gt, ncomp, out2, ws, n_samples=T, seed=seed)
    assert torch.equal(out, out2)


def test_residual_sampled_exact_sketch_is_zero(dev):
    """A = F G^T exactly representable: every sampled error is (FP32 dot rounding)^2 ~ 0."""
    from paper_1607_07395_b200.dist import make_plan
    m, n, r = 1000, 800, 4
    g = np.random.default_rng(1)
    F = g.integers(-3, 4, (m, r)).astype(np.float32)
    G = g.integers(-3, 4, (n, r)).astype(np.float32)
    A = (F @ G.T).astype(np.float32)  # small integers: exact in FP32, the dot is exact too
    plan = make_plan(m, n, 32)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    Ft, Gt = torch.zeros((m, 32), device=dev), torch.zeros((n, 32), device=dev)
    Ft[:, :r], Gt[:, :r] = torch.from_numpy(F).to(dev), torch.from_numpy(G).to(dev)
    C.cabs_residual(plan, torch.from_numpy(A).to(dev), Ft, None, Gt, r, out, ws, n_samples=100000, seed=2)
    assert out[0].item() == 0.0 and out[1].item() > 0


def test_rbf_residual_requires_samples(dev):
    from paper_1607_07395_b200.dist import make_plan
    src, _ = _rbf(100, 80, 16, 1, dev)
    plan = make_plan(100, 80, 32)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    F, G = torch.zeros((100, 32), device=dev), torch.zeros((80, 32), device=dev)
    with pytest.raises(C.CabsError):
        C.cabs_residual(plan, src, F, None, G, 4, torch.zeros(2, dtype=torch.float64, device=dev), ws)


@pytest.mark.parametrize("m,n,k,iters", [(20000, 10000, 60, 5), (6000, 4000, 100, 5)])
def test_e2e_rbf_scaled(dev, tmp_path, m, n, k, iters):
    """Algorithm 2 on the implicit source with the sampled residual, first-divergence parity."""
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    from tests.parity import check_e2e
    src, osrc = _rbf(m, n, 16, 0, dev)
    T = 1 << 21
    cfg = CabsConfig(k, k, iters, seed=0, residual_samples=T)
    pipe = CabsPipeline(src, m, n, cfg)
    pipe.run()
    g = pipe.results()
    ref = O.cabs_run(osrc, k, k, iters, seed=0, n_samples=T)
    check_e2e(C, O, osrc, g, ref, pipe, log_path=tmp_path / "rbf.json", n_samples=T)
