"""Pins for the oracle's k x k SVD and sketching routine (oracle/cabs.py).

P4 (SVD closed forms), P5 (Eq. 2 exact recovery), P6 (STABILIZED
closed forms), P11 (embedding identity), Z16 (index
permutation invariance).  F1: STABILIZED is not exact on exact-rank input.
"""
import math

import numpy as np
import pytest

from oracle import cabs as O


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------- P4: SVD
def test_svd_diag():
    Uw, s, Vw = O.svd_w(np.diag([2.0, 1.0]))
    assert np.allclose(s, [2.0, 1.0], rtol=0, atol=1e-15)


def test_svd_rank_one():
    W = np.outer([1.0, 2.0], [3.0, 4.0])
    Uw, s, Vw = O.svd_w(W)
    assert s.size == 1
    assert abs(s[0] - math.sqrt(5.0) * 5.0) < 1e-13
    assert np.allclose((Uw * s) @ Vw.T, W, atol=1e-13)


@pytest.mark.parametrize("shape", [(5, 3), (40, 40), (200, 200)])
def test_svd_reconstruction_orthogonality(shape):
    r = np.random.default_rng(shape[0])
    W = r.standard_normal(shape)
    Uw, s, Vw = O.svd_w(W)
    assert np.linalg.norm((Uw * s) @ Vw.T - W) < 1e-10 * np.linalg.norm(W)
    assert np.allclose(Uw.T @ Uw, np.eye(s.size), atol=1e-12)
    assert np.allclose(Vw.T @ Vw, np.eye(s.size), atol=1e-12)
    assert np.all(np.diff(s) <= 0)
    # sigma^2 are the eigenvalues of W^T W (independent routine)
    ev = np.sort(np.linalg.eigvalsh(W.T @ W))[::-1][: s.size]
    assert np.allclose(s**2, ev, rtol=1e-9, atol=1e-9 * ev[0])


def test_svd_canonical_signs():
    r = np.random.default_rng(3)
    Uw, s, Vw = O.svd_w(r.standard_normal((12, 12)))
    for i in range(s.size):
        p = int(np.argmax(np.abs(Uw[:, i])))
        assert Uw[p, i] > 0


def test_svd_truncation_tolerance():
    W = np.diag([1.0, 1e-6, 1e-13, 0.0])
    _, s, _ = O.svd_w(W, tol=1e-12)
    assert s.size == 2
    _, s, _ = O.svd_w(np.zeros((3, 3)))
    assert s.size == 0


def test_pinv_examples():
    # S:82-84 through the sketch's truncated pseudo-inverse
    C = np.eye(2); R = np.eye(2)
    assert np.allclose(O.pseudo_skeleton_dense(C, R, np.diag([2.0, 0.0])), np.diag([0.5, 0.0]))
    assert np.allclose(O.pseudo_skeleton_dense(C, R, np.diag([2.0, 4.0])), np.diag([0.5, 0.25]))


# ------------------------------------------------ P5: Eq. 2 exact recovery
def _lowrank(m, n, r, seed):
    g = np.random.default_rng(seed)
    return g.standard_normal((m, r)) @ g.standard_normal((r, n))


@pytest.mark.parametrize("m,n,k", [(40, 30, 5), (200, 150, 10), (600, 500, 20)])
def test_pseudo_skeleton_exact_recovery(m, n, k):
    A = _lowrank(m, n, k, m)
    g = np.random.default_rng(99)
    I = np.sort(g.choice(m, k, replace=False)); J = np.sort(g.choice(n, k, replace=False))
    C, R, W = O.gather(A, I, J)
    sk = O.sketch(C, R, W, m, n, k, mode=O.PSEUDO_SKELETON)
    assert _rel(sk.dense(), A) < 1e-9          # BASELINE north_star check #1
    r2, a2 = O.residual(A, sk.U, sk.V, sk.s)
    assert math.sqrt(r2 / a2) < 1e-9


def test_pseudo_skeleton_rank_one_spec():
    A = np.outer([1.0, 2.0], [1.0, 1.0, 1.0])
    C, R, W = O.gather(A, [0], [0])
    sk = O.sketch(C, R, W, 2, 3, 1, mode=O.PSEUDO_SKELETON)
    assert np.allclose(sk.dense(), A, atol=1e-15)


def test_pseudo_mode_equals_eq2_formula():
    g = np.random.default_rng(5)
    A = g.standard_normal((50, 40))
    I = np.sort(g.choice(50, 8, replace=False)); J = np.sort(g.choice(40, 8, replace=False))
    C, R, W = O.gather(A, I, J)
    sk = O.sketch(C, R, W, 50, 40, 8, mode=O.PSEUDO_SKELETON)
    assert _rel(sk.dense(), O.pseudo_skeleton_dense(C, R, W)) < 1e-10


def test_stabilized_not_exact_on_exact_rank():
    # F1: the stabilized routine is NOT an exact-recovery method.
    A = _lowrank(200, 150, 10, 7)
    g = np.random.default_rng(1)
    I = np.sort(g.choice(200, 10, replace=False)); J = np.sort(g.choice(150, 10, replace=False))
    sk = O.sketch(*O.gather(A, I, J), 200, 150, 10, mode=O.STABILIZED)
    assert _rel(sk.dense(), A) > 0.1


# ------------------------------------------------ P6: STABILIZED closed forms
def test_stabilized_full_sampling_collapse():
    g = np.random.default_rng(2)
    k = 7
    W = g.standard_normal((k, k))
    sk = O.sketch(W, W, W, k, k, k, mode=O.STABILIZED)
    assert _rel(sk.dense(), W) < 1e-13


def _block_replicated(row_sizes, col_sizes, k, seed):
    g = np.random.default_rng(seed)
    B = g.standard_normal((k, k))
    rl = np.repeat(np.arange(k), row_sizes)
    cl = np.repeat(np.arange(k), col_sizes)
    pr = g.permutation(rl.size); pc = g.permutation(cl.size)
    rl, cl = rl[pr], cl[pc]
    return B[np.ix_(rl, cl)], rl, cl


@pytest.mark.parametrize("mode", [O.STABILIZED, O.PSEUDO_SKELETON])
def test_block_replicated_exact(mode):
    k = 6
    A, rl, cl = _block_replicated([7] * k, [5] * k, k, 11)
    g = np.random.default_rng(4)
    I = np.sort([int(g.choice(np.where(rl == b)[0])) for b in range(k)])
    J = np.sort([int(g.choice(np.where(cl == b)[0])) for b in range(k)])
    sk = O.sketch(*O.gather(A, I, J), A.shape[0], A.shape[1], k, mode=mode)
    assert _rel(sk.dense(), A) < 1e-12              # 8.5e-16


def test_block_replicated_unequal_not_exact():
    k = 6
    A, rl, cl = _block_replicated([3, 5, 7, 9, 11, 13], [5] * k, k, 11)
    I = np.sort([int(np.where(rl == b)[0][0]) for b in range(k)])
    J = np.sort([int(np.where(cl == b)[0][0]) for b in range(k)])
    sk = O.sketch(*O.gather(A, I, J), A.shape[0], A.shape[1], k, mode=O.STABILIZED)
    assert _rel(sk.dense(), A) > 1e-3               # negative control (X9: 0.105)


def test_zero_singular_value_drops_component():
    g = np.random.default_rng(8)
    A = _lowrank(30, 20, 3, 8)
    I = np.sort(g.choice(30, 5, replace=False)); J = np.sort(g.choice(20, 5, replace=False))
    sk = O.sketch(*O.gather(A, I, J), 30, 20, 5)      # W has rank 3
    assert sk.r == 3
    assert np.all(np.isfinite(sk.U)) and np.all(np.isfinite(sk.V)) and np.all(np.isfinite(sk.s))


def test_extrapolated_norms_bounded_below_by_sigma():
    # C[I,:] = W, so ||C V_w e_i|| >= ||W V_w e_i|| = sigma_i: with a consistent triple the
    # zero-norm drop rule can never fire for a kept component.
    g = np.random.default_rng(14)
    A = g.standard_normal((70, 60))
    I = np.sort(g.choice(70, 10, replace=False)); J = np.sort(g.choice(60, 10, replace=False))
    sk = O.sketch(*O.gather(A, I, J), 70, 60, 10)
    assert np.all(sk.Nc >= sk.sigma * (1 - 1e-12)) and np.all(sk.Nr >= sk.sigma * (1 - 1e-12))


def test_zero_extrapolated_norm_dropped():
    # the safeguard itself, on an inconsistent triple whose C extrapolates to zero
    W = np.diag([2.0, 1.0])
    C = np.zeros((3, 2)); C[0, 0] = 1.0
    R = np.ones((2, 4))
    sk = O.sketch(C, R, W, 3, 4, 2)
    assert sk.r == 1 and np.all(np.isfinite(sk.U))


# ------------------------------------------------ P11, Z16
def test_embedding_identity():
    g = np.random.default_rng(9)
    A = g.standard_normal((60, 45))
    I = np.sort(g.choice(60, 9, replace=False)); J = np.sort(g.choice(45, 9, replace=False))
    sk = O.sketch(*O.gather(A, I, J), 60, 45, 9)
    P, Q = O.embeddings(sk)
    assert _rel(P @ Q.T, sk.dense()) < 1e-14


@pytest.mark.parametrize("mode", [O.STABILIZED, O.PSEUDO_SKELETON])
def test_permutation_invariance(mode):
    g = np.random.default_rng(12)
    A = g.standard_normal((300, 200))
    I = g.choice(300, 12, replace=False); J = g.choice(200, 12, replace=False)
    base = O.sketch(*O.gather(A, np.sort(I), np.sort(J)), 300, 200, 12, mode=mode).dense()
    pi, pj = g.permutation(12), g.permutation(12)
    other = O.sketch(*O.gather(A, np.sort(I)[pi], np.sort(J)[pj]), 300, 200, 12, mode=mode).dense()
    assert _rel(other, base) < 1e-12


def test_stabilized_scale_constant():
    # Z3: s = sigma * sqrt(m n)/k with k the sample count, not the kept rank
    g = np.random.default_rng(13)
    A = _lowrank(80, 50, 2, 13)
    I = np.sort(g.choice(80, 6, replace=False)); J = np.sort(g.choice(50, 6, replace=False))
    sk = O.sketch(*O.gather(A, I, J), 80, 50, 6)
    assert sk.r == 2
    assert np.allclose(sk.s, sk.sigma * math.sqrt(80 * 50) / 6, rtol=1e-15)


def test_gather_errors():
    A = np.arange(4.0).reshape(2, 2)
    assert O.gather(A, [1], [0, 1])[1].tolist() == [[2.0, 3.0]]
    assert O.gather(A, [0], [1])[2].tolist() == [[1.0]]
    with pytest.raises(IndexError):
        O.gather(A, [0, 0], [0])
    with pytest.raises(IndexError):
        O.gather(A, [2], [0])
