"""Pins for the residual (pin P10) and for Algorithm 2 end to end
(P14 exact CABS, P12 linear-access NaN poisoning, P13 transpose symmetry)."""
import math

import numpy as np
import pytest

from oracle import cabs as O
from oracle import rng


def test_residual_exact_and_zero_sketch():
    g = np.random.default_rng(0)
    F = g.standard_normal((30, 4)); G = g.standard_normal((20, 4))
    A = F @ G.T
    r2, a2 = O.residual(A, F, G)
    assert r2 < 1e-24 * a2
    r2, a2 = O.residual(A, F, G, s=np.zeros(4))
    assert r2 == a2 and O.relative_error(A, F, G, np.zeros(4)) == 1.0
    with pytest.raises(ZeroDivisionError):
        O.relative_error(np.zeros((3, 3)), np.ones((3, 1)), np.ones((3, 1)))


def test_residual_trace_identity():
    # ||A - F G^T||^2 = ||A||^2 - 2 tr(F^T A G) + tr((F^T F)(G^T G))  (independent formula)
    g = np.random.default_rng(1)
    A = g.standard_normal((37, 23)); F = g.standard_normal((37, 5)); G = g.standard_normal((23, 5))
    s = g.uniform(0.5, 2, 5)
    r2, a2 = O.residual(A, F, G, s, block=8)
    Fs = F * s
    ref = np.sum(A * A) - 2 * np.trace(Fs.T @ A @ G) + np.trace((Fs.T @ Fs) @ (G.T @ G))
    assert abs(r2 - ref) < 1e-10 * a2 and abs(a2 - np.sum(A * A)) < 1e-12 * a2


def _grouped_matrix(k, row_group_size, col_group_size, seed):
    g = np.random.default_rng(seed)
    B = g.standard_normal((k, k))
    rl = np.repeat(np.arange(k), row_group_size)[g.permutation(k * row_group_size)]
    cl = np.repeat(np.arange(k), col_group_size)[g.permutation(k * col_group_size)]
    return B[np.ix_(rl, cl)], rl, cl


@pytest.mark.parametrize("mode", [O.STABILIZED, O.PSEUDO_SKELETON])
def test_p14_end_to_end_exact(mode):
    """Block-replicated A with one pilot sample per block and an init of one point per
    group: the embeddings of a group coincide, Lloyd keeps one cluster per group, the snap
    of each group is its lowest index (exact ties), and the follow-up sketch is exact."""
    k = 5
    A, rl, cl = _grouped_matrix(k, 6, 4, 3)
    I = np.sort([int(np.where(rl == b)[0][-1]) for b in range(k)])
    J = np.sort([int(np.where(cl == b)[0][-1]) for b in range(k)])
    init_r = [int(np.where(rl == b)[0][1]) for b in range(k)]
    init_c = [int(np.where(cl == b)[0][1]) for b in range(k)]
    res = O.cabs_run(A, k, k, 4, mode=mode, I=I, J=J, init_rows=init_r, init_cols=init_c)
    exp_r = np.sort([int(np.where(rl == b)[0][0]) for b in range(k)])
    exp_c = np.sort([int(np.where(cl == b)[0][0]) for b in range(k)])
    assert np.array_equal(res.Ibar, exp_r) and np.array_equal(res.Jbar, exp_c)
    assert res.km_rows.objective[-1] < 1e-20 and res.km_cols.objective[-1] < 1e-20
    assert math.sqrt(res.resid_sq / res.a_sq) < 1e-12


def _lowrank_noisy(m, n, r, noise, seed):
    g = np.random.default_rng(seed)
    A = g.standard_normal((m, r)) @ (g.standard_normal((r, n)) / np.arange(1, r + 1)[:, None])
    return (A + noise * g.standard_normal((m, n))).astype(np.float32)


def test_p12_linear_access_nan_poison():
    A = _lowrank_noisy(120, 90, 6, 0.01, 4)
    res = O.cabs_run(A, 8, 8, 5, seed=3, with_residual=False)
    rows = np.union1d(res.I, res.Ibar); cols = np.union1d(res.J, res.Jbar)
    assert rows.size <= 16 and cols.size <= 16              # S:540 (2(k1+k2) bound, generous)
    Ap = np.full_like(A, np.nan)
    Ap[rows, :] = A[rows, :]
    Ap[:, cols] = A[:, cols]
    res2 = O.cabs_run(Ap, 8, 8, 5, seed=3, with_residual=False)
    for a, b in [(res.I, res2.I), (res.J, res2.J), (res.Ibar, res2.Ibar), (res.Jbar, res2.Jbar)]:
        assert np.array_equal(a, b)
    assert np.array_equal(res.follow.U, res2.follow.U) and np.array_equal(res.follow.s, res2.follow.s)
    assert np.all(np.isfinite(res2.follow.U)) and np.all(np.isfinite(res2.follow.V))


def test_p13_transpose_symmetry():
    A = _lowrank_noisy(70, 55, 5, 0.02, 6)
    k1, k2, it, seed = 7, 6, 6, 11
    res = O.cabs_run(A, k1, k2, it, seed=seed)
    init_r = rng.floyd(70, k2, seed, rng.TAG_INIT_ROWS)
    init_c = rng.floyd(55, k2, seed, rng.TAG_INIT_COLS)
    resT = O.cabs_run(np.ascontiguousarray(A.T), k1, k2, it, seed=seed, I=res.J, J=res.I,
                      init_rows=init_c, init_cols=init_r)
    assert np.array_equal(resT.Ibar, res.Jbar) and np.array_equal(resT.Jbar, res.Ibar)
    D, DT = res.follow.dense(), resT.follow.dense()
    assert np.linalg.norm(DT.T - D) < 1e-10 * np.linalg.norm(D)
    assert abs(resT.resid_sq - res.resid_sq) < 1e-10 * res.resid_sq


def test_cabs_run_deterministic_and_valid():
    A = _lowrank_noisy(200, 150, 10, 0.01, 8)
    a = O.cabs_run(A, 10, 10, 5, seed=1)
    b = O.cabs_run(A, 10, 10, 5, seed=1)
    assert np.array_equal(a.Ibar, b.Ibar) and a.resid_sq == b.resid_sq
    for idx, N in [(a.I, 200), (a.J, 150), (a.Ibar, 200), (a.Jbar, 150)]:
        assert np.all(np.diff(idx) > 0) and idx.min() >= 0 and idx.max() < N
    assert 0.0 < a.resid_sq < a.a_sq
    with pytest.raises(ValueError):
        O.cabs_run(A, 151, 10, 5)
