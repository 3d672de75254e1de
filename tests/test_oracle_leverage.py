"""Pins for the oracle's orthogonalization (Supp. section 3) and leverage-score
follow-up (P:312 variant (e)).

Orthogonalization: SPEC's examples (orthonormal input unchanged, scale shuffling), and the
thin SVD of the explicit product U diag(s) V^T (a textbook routine on the m x n matrix).
Sampling: the per-point uniforms, SPEC's examples, the first-draw multinomial and the
two-draw inclusion probabilities of successive sampling (brute-force formula), and the
exact-recovery end-to-end case."""
import itertools

import numpy as np
import pytest

from oracle import cabs as O
from oracle import rng


def _orthonormal(g, n, r):
    Q, _ = np.linalg.qr(g.standard_normal((n, r)))
    return Q


def test_uniform01_range_and_bits():
    u = rng.uniform01(7, rng.TAG_LEVERAGE_ROWS, np.arange(200000))
    assert np.all(u > 0) and np.all(u < 1)
    assert np.unique(u).size == u.size
    assert abs(u.mean() - 0.5) < 5 * np.sqrt(1 / 12 / u.size)
    # 53 bits: u * 2^53 - 1/2 is an integer
    x = u * 2.0 ** 53 - 0.5
    assert np.array_equal(x, np.floor(x))
    # the scalar Philox reference on one point (vectorised vs scalar implementation)
    w = rng.philox4x32_10((12345, 0, rng.TAG_LEVERAGE_COLS, 1), rng.seed_key(99))
    want = ((w[0] >> 5) * 67108864.0 + (w[1] >> 6) + 0.5) * 2.0 ** -53
    assert rng.uniform01(99, rng.TAG_LEVERAGE_COLS, [12345])[0] == want
    # streams differ by tag and seed
    assert not np.array_equal(u[:100], rng.uniform01(7, rng.TAG_LEVERAGE_COLS, np.arange(100)))
    assert not np.array_equal(u[:100], rng.uniform01(8, rng.TAG_LEVERAGE_ROWS, np.arange(100)))


def test_orthogonalize_orthonormal_input_unchanged():
    g = np.random.default_rng(1)
    U, V = _orthonormal(g, 40, 5), _orthonormal(g, 30, 5)
    s = np.array([5.0, 4.0, 3.0, 2.0, 1.0])
    Uo, so, Vo = O.orthogonalize(U, s, V)
    assert np.allclose(so, s, rtol=1e-10)
    assert np.allclose(Uo @ np.diag(so) @ Vo.T, U @ np.diag(s) @ V.T, atol=1e-12)


def test_orthogonalize_scale_shuffling():
    g = np.random.default_rng(2)
    U, V = g.standard_normal((50, 6)), g.standard_normal((35, 6))
    s = g.uniform(0.5, 2.0, 6)
    a = O.orthogonalize(U, s, V)
    b = O.orthogonalize(2 * U, s / 2, V)
    assert np.allclose(a[1], b[1], rtol=1e-12)
    assert np.allclose(a[0] @ np.diag(a[1]) @ a[2].T, b[0] @ np.diag(b[1]) @ b[2].T, atol=1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_orthogonalize_is_the_thin_svd_of_the_product(seed):
    g = np.random.default_rng(10 + seed)
    m, n, r = 60, 45, 7
    U, V = g.standard_normal((m, r)), g.standard_normal((n, r))
    s = g.uniform(0.1, 3.0, r)
    Uo, so, Vo = O.orthogonalize(U, s, V)
    M = U @ np.diag(s) @ V.T
    Ur, sr, Vrt = np.linalg.svd(M)
    assert np.allclose(so, sr[:r], rtol=1e-12)
    assert np.allclose(Uo.T @ Uo, np.eye(r), atol=1e-12) and np.allclose(Vo.T @ Vo, np.eye(r), atol=1e-12)
    assert np.allclose(np.abs(np.sum(Uo * Ur[:, :r], axis=0)), 1.0, atol=1e-10)  # same vectors up to sign
    assert np.allclose(Uo @ np.diag(so) @ Vo.T, M, atol=1e-12 * np.abs(M).max())


def test_leverage_scores_and_spec_examples():
    F = np.zeros((6, 2))
    F[0, 0] = F[1, 1] = 1.0  # rows e1, e2
    assert O.leverage_scores(F).tolist() == [0.5, 0.5, 0, 0, 0, 0]
    for seed in range(5):
        assert O.leverage_sample(F, 2, seed, rng.TAG_LEVERAGE_ROWS).tolist() == [0, 1]
    with pytest.raises(ValueError):
        O.leverage_sample(F, 3, 0, rng.TAG_LEVERAGE_ROWS)
    g = np.random.default_rng(3)
    Q = _orthonormal(g, 80, 6)
    assert abs(O.leverage_scores(Q).sum() - 1.0) < 1e-12


def test_first_draw_is_proportional_to_scores():
    """scores [0.5, 0.25, 0.25], k = 1 -> frequencies within 5 sigma."""
    F = np.sqrt(np.array([[0.5], [0.25], [0.25]]))
    T = 3000
    cnt = np.zeros(3)
    for seed in range(T):
        cnt[O.leverage_sample(F, 1, seed, rng.TAG_LEVERAGE_ROWS)[0]] += 1
    p = np.array([0.5, 0.25, 0.25])
    assert np.all(np.abs(cnt / T - p) < 5 * np.sqrt(p * (1 - p) / T))


def test_two_draw_inclusion_matches_successive_sampling():
    """Without replacement, proportional to the scores: P(i in S) for k = 2 by the
    brute-force successive-sampling formula, within 5 sigma over independent streams."""
    w = np.array([0.4, 0.3, 0.2, 0.1])
    F = np.sqrt(w)[:, None]
    incl = np.zeros(4)
    for i, j in itertools.permutations(range(4), 2):
        pr = w[i] / w.sum() * w[j] / (w.sum() - w[i])
        incl[i] += pr
        incl[j] += pr
    T = 4000
    cnt = np.zeros(4)
    for seed in range(T):
        for l in O.leverage_sample(F, 2, seed, rng.TAG_LEVERAGE_COLS):
            cnt[l] += 1
    assert np.all(np.abs(cnt / T - incl) < 5 * np.sqrt(incl * (1 - incl) / T))


def test_equal_scores_give_uniform_inclusion():
    F = np.full((10, 1), np.sqrt(0.1))
    T, k = 3000, 3
    cnt = np.zeros(10)
    for seed in range(T):
        cnt[O.leverage_sample(F, k, seed, rng.TAG_LEVERAGE_ROWS)] += 1
    p = k / 10
    assert np.all(np.abs(cnt / T - p) < 5 * np.sqrt(p * (1 - p) / T))


def test_followup_leverage_exact_low_rank():
    g = np.random.default_rng(7)
    m, n, r, k = 60, 45, 4, 8
    A = g.standard_normal((m, r)) @ g.standard_normal((n, r)).T
    res = O.cabs_run(A, 10, k, 5, seed=3, mode=O.PSEUDO_SKELETON, followup="leverage")
    Uo, so, Vo = O.orthogonalize(res.pilot.U, res.pilot.s, res.pilot.V)
    assert res.Ibar.tolist() == O.leverage_sample(Uo, k, 3, rng.TAG_LEVERAGE_ROWS).tolist()
    assert res.Jbar.tolist() == O.leverage_sample(Vo, k, 3, rng.TAG_LEVERAGE_COLS).tolist()
    assert np.sqrt(res.resid_sq / res.a_sq) < 1e-9
