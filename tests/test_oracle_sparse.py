"""Pins of the oracle's sparse source ("For sparse matrices",
Table 1; SPEC S:23-28 SparseMat) and of its split residual (the P:313 error as
nonzeros + r x r Gram products).

Each pin is fixed outside the oracle's own formulas: SPEC's worked example, a dense
matrix assembled independently by scipy.sparse, the identity ||A - B||^2 = ||A||^2 - 2<A,B> +
||B||^2 checked against the dense definition on random cases (a dropped factor 2, a missing s or
a transposed Gram product fails it), closed-form cases, the equality of the whole CABS run on the
sparse source and on its dense copy (every step depends on A only through its entries), exact
recovery of a sparse rank-2 matrix (Eq. 2), and the workload's density."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import cabs as O


def _random_csr(m, n, density, seed, rank=None):
    g = np.random.default_rng(seed)
    M = sp.random(m, n, density=density, random_state=seed, format="csr", dtype=np.float64)
    if rank is not None:  # values of a low-rank product at the kept positions
        L = g.standard_normal((m, rank)) @ g.standard_normal((rank, n))
        M.data = L[M.nonzero()].astype(np.float32).astype(np.float64)
    M.sort_indices()
    return O.CsrSource(M.indptr, M.indices, M.data, M.shape), M


def test_spec_coordinate_example():
    # coordinate entries (1,1,5.0),(2,2,3.0) of a 2 x 2 matrix -> diag(5, 3) (1-based)
    src = O.CsrSource([0, 1, 2], [0, 1], [5.0, 3.0], (2, 2))
    assert np.array_equal(src.dense(), np.diag([5.0, 3.0]))
    assert src.nnz == 2


def test_entries_match_scipy_dense():
    src, M = _random_csr(37, 53, 0.1, 1)
    D = M.toarray()
    assert np.array_equal(src.dense(), D)
    I, J = np.array([3, 0, 36]), np.array([52, 7, 8, 0])
    assert np.array_equal(src.entries(I, J), D[np.ix_(I, J)])
    C, R, W = O.gather(src, I, J)
    assert np.array_equal(C, D[:, J]) and np.array_equal(R, D[I, :]) and np.array_equal(W, D[np.ix_(I, J)])


def test_invariants_enforced():
    with pytest.raises(ValueError):
        O.CsrSource([0, 2], [3, 3], [1.0, 2.0], (1, 5))     # duplicate (row, col)
    with pytest.raises(ValueError):
        O.CsrSource([0, 2], [3, 1], [1.0, 2.0], (1, 5))     # not sorted
    with pytest.raises(IndexError):
        O.CsrSource([0, 1], [5], [1.0], (1, 5))             # column out of range


@pytest.mark.parametrize("m,n,density,r,use_s,seed", [(40, 30, 0.2, 3, True, 0), (100, 70, 0.05, 8, False, 1),
                                                      (25, 90, 0.3, 1, True, 2), (60, 60, 0.0, 4, True, 3)])
def test_residual_split_equals_definition(m, n, density, r, use_s, seed):
    src, M = _random_csr(m, n, density, seed)
    g = np.random.default_rng(seed + 10)
    F = g.standard_normal((m, r))
    G = g.standard_normal((n, r))
    s = g.uniform(0.5, 2.0, r) if use_s else None
    r2, a2 = O.residual_sparse(src, F, G, s)
    B = (F * (s if use_s else 1.0)) @ G.T
    D = M.toarray()
    assert abs(a2 - np.sum(D * D)) <= 1e-12 * max(1.0, np.sum(D * D))
    assert abs(r2 - np.sum((D - B) ** 2)) <= 1e-10 * np.sum((D - B) ** 2)
    # the oracle's plain definition on the sparse source agrees as well
    rr2, ra2 = O.residual(src, F, G, s)
    assert abs(rr2 - r2) <= 1e-10 * rr2 and abs(ra2 - a2) <= 1e-12 * max(1.0, ra2)


def test_residual_split_closed_forms():
    # A = e_0 e_1^T (one nonzero 2 at (0, 1)); F = e_0, G = e_1, s = [3]: ||A - 3 e0 e1^T||^2 = 1
    src = O.CsrSource([0, 1, 1], [1], [2.0], (2, 3))
    F = np.array([[1.0], [0.0]])
    G = np.array([[0.0], [1.0], [0.0]])
    r2, a2 = O.residual_sparse(src, F, G, [3.0])
    assert r2 == 1.0 and a2 == 4.0
    # an all-zero A: the error is ||F S G^T||^2 = (sum F^2)(sum G^2) s^2 for rank 1
    z = O.CsrSource([0, 0, 0], [], [], (2, 3))
    F = np.array([[1.0], [2.0]])
    G = np.array([[1.0], [1.0], [3.0]])
    r2, a2 = O.residual_sparse(z, F, G, [0.5])
    assert a2 == 0.0 and abs(r2 - 5.0 * 11.0 * 0.25) < 1e-12


def test_cabs_run_on_sparse_equals_dense_copy():
    src, M = _random_csr(300, 240, 0.05, 4, rank=6)
    D = M.toarray()
    a = O.cabs_run(src, 12, 10, 5, seed=3, weight_kind=O.WEIGHT_POWER)
    b = O.cabs_run(D, 12, 10, 5, seed=3, weight_kind=O.WEIGHT_POWER)
    assert np.array_equal(a.I, b.I) and np.array_equal(a.J, b.J)
    assert np.array_equal(a.Ibar, b.Ibar) and np.array_equal(a.Jbar, b.Jbar)
    assert np.array_equal(a.follow.U, b.follow.U) and np.array_equal(a.follow.s, b.follow.s)
    assert a.resid_sq == b.resid_sq
    r2, a2 = O.residual_sparse(src, a.follow.U, a.follow.V, a.follow.s)
    assert abs(r2 - a.resid_sq) <= 1e-9 * a.a_sq and abs(a2 - a.a_sq) <= 1e-12 * a.a_sq


def test_sparse_rank2_exact_recovery():
    # A = u1 v1^T + u2 v2^T with sparse u, v (zeros outside half the rows / columns): rank 2.
    # With every row and column sampled the pilot W = A has rank 2 and the pseudo-skeleton
    # C W^+ R reproduces A exactly (Eq. 2).
    g = np.random.default_rng(7)
    m, n = 30, 24
    U = g.standard_normal((m, 2)) * (g.random((m, 2)) < 0.5)
    V = g.standard_normal((n, 2)) * (g.random((n, 2)) < 0.5)
    D = U @ V.T
    M = sp.csr_matrix(D)
    M.sort_indices()
    src = O.CsrSource(M.indptr, M.indices, M.data, M.shape)
    res = O.cabs_run(src, min(m, n), 2, 3, seed=1, I=np.arange(min(m, n)), J=np.arange(min(m, n)),
                     mode=O.PSEUDO_SKELETON)
    assert res.pilot.r == 2
    Ap = res.pilot.dense()
    assert np.abs(Ap - D).max() <= 1e-9 * max(1.0, np.abs(D).max())


def test_workload_density_and_structure():
    # sparse_lowrank density 0.0056 -> nonzero fraction within +-10% of 0.0056
    import torch  # noqa: F401
    from workloads import SPARSE_CONFIGS, csr_to_csc, make_sparse, scaled
    cfg = scaled(SPARSE_CONFIGS["s1"], 3000, 4600)
    ip, ix, v = make_sparse(cfg, 0.0056)
    frac = int(ip[-1]) / (cfg.m * cfg.n)
    assert abs(frac - 0.0056) <= 0.1 * 0.0056
    src = O.CsrSource(ip.numpy(), ix.numpy(), v.numpy(), (cfg.m, cfg.n))  # validates sorting / duplicates
    cp, ri, cv = csr_to_csc(ip, ix, v, cfg.n)
    T = sp.csc_matrix((cv.numpy().astype(np.float64), ri.numpy(), cp.numpy()), shape=(cfg.m, cfg.n))
    J = np.array([0, 17, 4599])
    assert np.array_equal(T[:, J].toarray(), src.entries(np.arange(cfg.m), J))
    assert math.isfinite(float(v.abs().max()))
