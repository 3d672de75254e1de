"""Pins of the oracle's implicit RBF source and sampled residual (BASELINE.json configs[4];
PAPER.md P:24, P:29 entries generated on access, P:313 the error metric; readings Z17 / Z23).

Each pin is fixed by mathematics, not by the oracle's own formula: closed-form kernel values,
positive semi-definiteness of a Gaussian Gram matrix, the exact equality of the estimator with
the dense residual when the pairs enumerate every entry once, unbiasedness over seeds, and the
uniformity / range / determinism of the Philox pair stream (Philox and Lemire themselves are
pinned in test_oracle_rng.py)."""
import math

import numpy as np
import pytest

from oracle import cabs as O
from oracle import rng


def test_rbf_closed_forms():
    sigma = 1.7
    x = np.zeros((3, 4))
    x[1, 0] = math.sqrt(2.0) * sigma            # |x1 - x0|^2 = 2 sigma^2  -> e^-1
    x[2, :] = [sigma, sigma, sigma, 0.0]        # |x2 - x0|^2 = 3 sigma^2  -> e^-1.5
    A = O.RbfSource(x, x, sigma).entries(np.arange(3), np.arange(3))
    assert np.allclose(np.diag(A), 1.0, rtol=0, atol=0)
    assert abs(A[0, 1] - math.exp(-1.0)) < 1e-15 and abs(A[1, 0] - math.exp(-1.0)) < 1e-15
    assert abs(A[0, 2] - math.exp(-1.5)) < 1e-15
    # |x1 - x2|^2 = (sqrt2 - 1)^2 s^2 + 2 s^2
    assert abs(A[1, 2] - math.exp(-((math.sqrt(2) - 1) ** 2 + 2) / 2)) < 1e-15


def test_rbf_gram_is_psd_and_symmetric():
    g = np.random.default_rng(0)
    x = g.standard_normal((60, 16)).astype(np.float32)
    src = O.RbfSource(x, x, 2.0)
    K = src.entries(np.arange(60), np.arange(60))
    assert np.array_equal(K, K.T)
    assert np.linalg.eigvalsh(K).min() > -1e-10  # Gaussian kernel: positive (semi)definite
    assert np.all((K > 0) & (K <= 1))


def test_rbf_at_matches_grid_and_gather():
    g = np.random.default_rng(1)
    src = O.RbfSource(g.standard_normal((30, 16)), g.standard_normal((20, 16)), 3.0)
    i, j = g.integers(0, 30, 100), g.integers(0, 20, 100)
    grid = src.entries(np.arange(30), np.arange(20))
    assert np.array_equal(src.at(i, j), grid[i, j])
    C, R, W = O.gather(src, [3, 7], [1, 2, 19])
    assert np.array_equal(C, grid[:, [1, 2, 19]]) and np.array_equal(R, grid[[3, 7]])
    assert np.array_equal(W, grid[np.ix_([3, 7], [1, 2, 19])])


def test_pairs_range_determinism_uniformity():
    i, j = rng.residual_pairs(7, 70000, 7, 5)
    assert i.min() >= 0 and i.max() < 7 and j.min() >= 0 and j.max() < 5
    i2, j2 = rng.residual_pairs(7, 70000, 7, 5)
    assert np.array_equal(i, i2) and np.array_equal(j, j2)
    i3, _ = rng.residual_pairs(8, 70000, 7, 5)
    assert not np.array_equal(i, i3)
    # chi-square over the 35 cells (34 dof): mean 34, sd ~8.2; 5 sd bound
    cnt = np.bincount(i * 5 + j, minlength=35)
    chi2 = float(np.sum((cnt - 2000.0) ** 2 / 2000.0))
    assert chi2 < 34 + 5 * math.sqrt(68)
    # a window of the stream equals the same pairs drawn from the start
    iw, jw = rng.residual_pairs(7, 100, 7, 5, t0=500)
    assert np.array_equal(iw, i[500:600]) and np.array_equal(jw, j[500:600])


def test_pairs_rejection_heavy_bound_is_uniform():
    """s = 2^31 + 1 rejects about half of all words: the multi-word / multi-attempt path is
    exercised on most pairs; the draws stay uniform over 16 equal buckets."""
    s = (1 << 31) + 1
    i, j = rng.residual_pairs(3, 40000, s, s)
    assert i.max() < s and j.max() < s and i.min() >= 0
    for v in (i, j):
        cnt = np.bincount((v * 16) // s, minlength=16)
        chi2 = float(np.sum((cnt - 2500.0) ** 2 / 2500.0))
        assert chi2 < 15 + 5 * math.sqrt(30)


def test_sampled_residual_enumerating_pairs_equals_dense():
    g = np.random.default_rng(2)
    m, n, r = 13, 9, 3
    A = g.standard_normal((m, n))
    F, G, s = g.standard_normal((m, r)), g.standard_normal((n, r)), g.uniform(0.5, 2, r)
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    perm = g.permutation(m * n)
    est = O.residual_sampled(A, F, G, ii.ravel()[perm], jj.ravel()[perm], s)
    exact = O.residual(A, F, G, s)
    assert abs(est[0] - exact[0]) <= 1e-12 * exact[0] and abs(est[1] - exact[1]) <= 1e-12 * exact[1]
    # the same for the implicit source
    src = O.RbfSource(g.standard_normal((m, 4)), g.standard_normal((n, 4)), 1.5)
    est = O.residual_sampled(src, F, G, ii.ravel(), jj.ravel(), s)
    exact = O.residual(src, F, G, s)
    assert abs(est[0] - exact[0]) <= 1e-12 * exact[0] and abs(est[1] - exact[1]) <= 1e-12 * exact[1]


def test_sampled_residual_exact_sketch_and_constant_matrix():
    g = np.random.default_rng(3)
    F, G = g.standard_normal((40, 4)), g.standard_normal((30, 4))
    A = F @ G.T
    i, j = rng.residual_pairs(1, 500, 40, 30)
    r2, a2 = O.residual_sampled(A, F, G, i, j)
    assert r2 < 1e-20 * a2
    # constant A = c, zero sketch: every estimate equals m n c^2 exactly (any pairs)
    c = 0.75
    r2, a2 = O.residual_sampled(np.full((40, 30), c), np.zeros((40, 4)), np.zeros((30, 4)), i, j)
    assert r2 == a2 == pytest.approx(40 * 30 * c * c, rel=1e-15)


def test_sampled_residual_unbiased():
    """E[estimate] = the dense value: the mean over 3000 seeds is within 5 standard errors."""
    g = np.random.default_rng(4)
    m, n = 4, 3
    A = g.standard_normal((m, n))
    F, G = g.standard_normal((m, 1)), g.standard_normal((n, 1))
    exact_r2, exact_a2 = O.residual(A, F, G)
    T = 6
    est = np.array([O.residual_sampled(A, F, G, *rng.residual_pairs(seed, T, m, n)) for seed in range(3000)])
    for col, exact in ((0, exact_r2), (1, exact_a2)):
        mean, se = est[:, col].mean(), est[:, col].std(ddof=1) / math.sqrt(est.shape[0])
        assert abs(mean - exact) < 5 * se, (col, mean, exact, se)


def test_cabs_run_on_rbf_source_small():
    """Algorithm 2 on the implicit source equals Algorithm 2 on its materialised matrix."""
    from workloads import CONFIGS, make_rbf, scaled
    cfg = scaled(CONFIGS["c5"], 600, 400, 20, 20, 3)
    x, y, sigma = make_rbf(cfg)
    src = O.RbfSource(x.numpy(), y.numpy(), sigma)
    dense = src.entries(np.arange(600), np.arange(400))
    a = O.cabs_run(src, 20, 20, 3, seed=0, n_samples=5000)
    b = O.cabs_run(dense, 20, 20, 3, seed=0, n_samples=5000)
    assert np.array_equal(a.Ibar, b.Ibar) and np.array_equal(a.Jbar, b.Jbar)
    assert a.resid_sq == b.resid_sq and a.a_sq == b.a_sq
    # the sampled estimate is near the dense value on this smooth matrix
    r2, a2 = O.residual(src, a.follow.U, a.follow.V, a.follow.s)
    assert abs(a.a_sq - a2) < 0.05 * a2


def test_sampled_residual_row_remap_equals_full_factor():
    """f_rows (F given only on the sampled rows) is a re-indexing: identical result."""
    g = np.random.default_rng(5)
    src = O.RbfSource(g.standard_normal((50, 16)), g.standard_normal((40, 16)), 4.0)
    F, G, s = g.standard_normal((50, 3)), g.standard_normal((40, 3)), g.uniform(0.5, 2, 3)
    i, j = rng.residual_pairs(3, 2000, 50, 40)
    iu, inv = np.unique(i, return_inverse=True)
    assert O.residual_sampled(src, F, G, i, j, s) == O.residual_sampled(src, F[iu], G, i, j, s, f_rows=inv)
