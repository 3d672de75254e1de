"""Pins of the oracle's NEXT-4 baselines: BR-CUR (Algorithm 1),
Sketch-CUR (P:115, P:312 (a)) and the rank sweep on a validation set.

Fixed outside the oracle's own formulas: the four Penrose conditions of the pseudo-inverse;
SPEC's worked examples (S:256-258 projector identity and the pseudo-skeleton equivalence of
coincident base / target sampling, S:264-266 Sketch-CUR sizes and exact recovery, S:357-358 the
validation sweep); least-squares optimality of U* against random perturbations; exact recovery
of a rank-r matrix; the sweep's end points (the holdout energy at rank 0, zero error once the
rank of an exact sketch is reached)."""
import numpy as np
import pytest

from oracle import cabs as O
from oracle import rng


def _lowrank(m, n, r, seed):
    g = np.random.default_rng(seed)
    return g.standard_normal((m, r)) @ g.standard_normal((r, n))


@pytest.mark.parametrize("shape,rank", [((7, 5), 5), ((6, 9), 3), ((12, 12), 12), ((10, 4), 1)])
def test_pinv_penrose(shape, rank):
    X = _lowrank(shape[0], shape[1], rank, sum(shape) + rank)
    P = O.pinv(X)
    assert np.allclose(X @ P @ X, X, atol=1e-10 * np.abs(X).max())
    assert np.allclose(P @ X @ P, P, atol=1e-10 * np.abs(P).max())
    assert np.allclose((X @ P).T, X @ P, atol=1e-10)
    assert np.allclose((P @ X).T, P @ X, atol=1e-10)


def test_br_cur_all_indices_reproduce_a():
    # base = target = all indices on a 6 x 5 full-rank matrix -> C U R = A A^+ A A^+ A = A
    A = np.random.default_rng(1).standard_normal((6, 5))
    res = O.br_cur(A, np.arange(6), np.arange(5), np.arange(6), np.arange(5))
    assert np.abs(res.dense() - A).max() < 1e-8


def test_br_cur_coincident_sampling_is_pseudo_skeleton():
    # S:258 (section 2.2 item 2): base = target -> C W^+ R
    A = _lowrank(8, 6, 2, 2)
    I, J = np.array([1, 5]), np.array([0, 4])
    res = O.br_cur(A, I, J, I, J)
    C, R, W = O.gather(A, I, J)
    assert np.abs(res.dense() - O.pseudo_skeleton_dense(C, R, W)).max() < 1e-8


def test_br_cur_middle_is_least_squares_optimal():
    g = np.random.default_rng(3)
    A = g.standard_normal((40, 30))
    Ibr, Ibc = np.array([2, 7, 11, 20]), np.array([0, 3, 9, 29])
    Itr, Itc = np.arange(0, 40, 3), np.arange(1, 30, 3)
    res = O.br_cur(A, Ibr, Ibc, Itr, Itc)
    Cb, Rb, M = res.C[Itr], res.R[:, Itc], A[np.ix_(Itr, Itc)]
    best = np.linalg.norm(M - Cb @ res.U @ Rb)
    for _ in range(100):
        D = 1e-3 * g.standard_normal(res.U.shape)
        assert np.linalg.norm(M - Cb @ (res.U + D) @ Rb) >= best - 1e-12


def test_br_cur_exact_recovery_and_empty_target():
    A = _lowrank(50, 40, 4, 4)
    res = O.br_cur(A, [0, 10, 20, 30, 45], [1, 8, 15, 22, 39], np.arange(0, 50, 4), np.arange(0, 40, 4))
    assert np.abs(res.dense() - A).max() < 1e-8 * np.abs(A).max()
    with pytest.raises(ValueError):
        O.br_cur(A, [0], [0], [], [1])


def test_sketch_cur_sizes_and_recovery():
    A = _lowrank(30, 30, 2, 5)
    res, Itr, Itc = O.sketch_cur(A, np.array([3, 17]), np.array([4, 21]), 3, seed=0)
    assert Itr.size == 6 and Itc.size == 6
    assert np.array_equal(Itr, rng.floyd(30, 6, 0, rng.TAG_TARGET_ROWS))
    ok = 0
    for seed in range(50):
        g = np.random.default_rng(100 + seed)
        Ib = np.sort(g.choice(30, 2, replace=False))
        Jb = np.sort(g.choice(30, 2, replace=False))
        res, _, _ = O.sketch_cur(A, Ib, Jb, 3, seed=seed)
        ok += np.linalg.norm(res.dense() - A) / np.linalg.norm(A) < 1e-6
    assert ok >= 45
    with pytest.raises(ValueError):
        O.sketch_cur(A, np.arange(11), np.arange(11), 3, seed=0)  # 33 > 30


def test_holdout_errors_end_points_and_exact_rank():
    # an exact rank-3 matrix and an exact sketch (pseudo-skeleton, all 6 sampled rows / columns)
    A = _lowrank(60, 50, 3, 6)
    I, J = np.arange(0, 60, 10), np.arange(0, 50, 8)[:6]
    sk = O.sketch(*O.gather(A, I, J), 60, 50, 6, mode=O.PSEUDO_SKELETON)
    Hr = O.holdout_indices(60, 12, 0, rng.TAG_HOLDOUT_ROWS, I)
    Hc = O.holdout_indices(50, 12, 0, rng.TAG_HOLDOUT_COLS, J)
    assert not np.isin(Hr, I).any() and not np.isin(Hc, J).any() and np.all(np.diff(Hr) > 0)
    e = O.holdout_errors(A, sk.U, sk.s, sk.V, Hr, Hc)
    assert e.size == sk.r + 1
    assert abs(e[0] - np.sum(A[np.ix_(Hr, Hc)] ** 2)) <= 1e-12 * e[0]
    assert sk.r == 3 and e[3] < 1e-16 * e[0]                      # exact at the rank of A
    rho = O.validate_rank(e)                                      # lowest rank within 1e-8 of the floor
    assert e[rho] <= e[1:].min() + 1e-8 * e[0] and rho <= 3
    assert O.validate_rank([5.0, 2.0]) == 1                       # k = 1 -> 1
    assert O.validate_rank([5.0, 2.0, 1.0, 1.0]) == 2             # ties -> lowest rank


def test_holdout_errors_gram_expansion_identity():
    # the expansion the GPU evaluates: e[rho] = ||B||^2 - 2 sum_{t<=rho} s_t u_t^T B v_t
    #   + sum_{t,t'<=rho} s_t s_t' (U_H^T U_H)_{tt'} (V_H^T V_H)_{tt'}
    g = np.random.default_rng(8)
    A = g.standard_normal((40, 30))
    U, V, s = g.standard_normal((40, 7)), g.standard_normal((30, 7)), g.uniform(0.5, 2, 7)
    Hr, Hc = np.array([0, 3, 5, 9, 22]), np.array([1, 2, 8, 29])
    e = O.holdout_errors(A, U, s, V, Hr, Hc)
    B = A[np.ix_(Hr, Hc)]
    Uh, Vh = U[Hr], V[Hc]
    a = np.einsum("it,ij,jt->t", Uh, B, Vh)
    G = (Uh.T @ Uh) * (Vh.T @ Vh) * np.outer(s, s)
    for rho in range(8):
        x = np.sum(B * B) - 2 * np.sum(s[:rho] * a[:rho]) + np.sum(G[:rho, :rho])
        assert abs(x - e[rho]) <= 1e-10 * e[0]
