"""FP64 oracle of the CABS hot path (TEST INFRASTRUCTURE ONLY).

Plain, slow, obviously-correct NumPy float64 code that follows the paper step by
step (Algorithm 2; the sketching routine of §4.1,
P:222-232; weighted k-means, Eq. 6).  Where a step has a plain
definition (gathers, nearest-centre argmin, the Frobenius residual) the oracle
computes that definition directly.  Where the paper is silent we follow the
readings Z1-Z25 listed in DESIGN.md ("Readings of the paper").

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference leg may import this module.  It shares no code with the CUDA path.

Parity status per function:
  gather, svd_w, sketch, embeddings, argmin_with_gap, lloyd, snap, residual, cabs_run,
  row_sq_norms, hard_threshold_select, hard_threshold_followup, orthogonalize,
  leverage_scores, leverage_sample, RbfSource, residual_sampled, CsrSource, residual_sparse,
  pinv, br_cur, sketch_cur, holdout_indices, holdout_errors, validate_rank: pinned
  (tests/test_oracle_*.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import rng

STABILIZED = 0
PSEUDO_SKELETON = 1

WEIGHT_CONST = 0
WEIGHT_POWER = 1

DEFAULT_TOL = 1e-12  # keep sigma_i > tol * sigma_1
NEAR_TIE_GAP = 1e-5  # BASELINE.json north_star: relative distance gap < 1e-5


# --------------------------------------------------------------------------
# Step 1 / step 3 gathers:  C = A[:, J], R = A[I, :], W = A[I, J]
# --------------------------------------------------------------------------
def check_indices(idx, N, what="index"):
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() >= N):
        raise IndexError(f"{what} out of range [0, {N})")
    if np.unique(idx).size != idx.size:
        raise IndexError(f"duplicate {what}")
    return idx


class RbfSource:
    """The implicit c5 matrix (BASELINE.json configs[4]): A_ij = exp(-||x_i - y_j||^2 / (2 sigma^2)),
    entries generated on access ("never knowing the remaining entries").
    x (m x d), y (n x d) are the FP32 points; sigma is given (an input of the workload)."""

    def __init__(self, x, y, sigma):
        self.x = np.asarray(x, np.float64)
        self.y = np.asarray(y, np.float64)
        self.sigma = float(sigma)
        self.shape = (self.x.shape[0], self.y.shape[0])

    def entries(self, I, J):
        """A[I][:, J] as float64: the definition, ||x_i - y_j||^2 summed over the d coordinates."""
        X = self.x[np.asarray(I, np.int64)]
        Y = self.y[np.asarray(J, np.int64)]
        d2 = np.zeros((X.shape[0], Y.shape[0]))
        for l in range(X.shape[1]):
            diff = X[:, l][:, None] - Y[:, l][None, :]
            d2 += diff * diff
        return np.exp(-d2 / (2.0 * self.sigma ** 2))

    def at(self, i, j):
        """A_{i_t j_t} for position arrays i, j (elementwise)."""
        X = self.x[np.asarray(i, np.int64)]
        Y = self.y[np.asarray(j, np.int64)]
        d2 = np.zeros(X.shape[0])
        for l in range(X.shape[1]):  # the same coordinate order as entries()
            diff = X[:, l] - Y[:, l]
            d2 += diff * diff
        return np.exp(-d2 / (2.0 * self.sigma ** 2))


class CsrSource:
    """A sparse A ("For sparse matrices"; Table 1 P:301-302 sparsity column;
    SPEC S:23-28 SparseMat) in compressed sparse row form: the nonzeros of row i are
    data[indptr[i]:indptr[i+1]] at columns indices[indptr[i]:indptr[i+1]] (strictly increasing,
    no duplicates).  Every other entry is 0."""

    def __init__(self, indptr, indices, data, shape):
        self.indptr = np.asarray(indptr, np.int64)
        self.indices = np.asarray(indices, np.int64)
        self.data = np.asarray(data, np.float64)
        self.shape = (int(shape[0]), int(shape[1]))
        m, n = self.shape
        if self.indptr.shape != (m + 1,) or self.indptr[0] != 0 or np.any(np.diff(self.indptr) < 0):
            raise ValueError("bad indptr")
        if self.indices.size != self.indptr[-1] or self.data.size != self.indices.size:
            raise ValueError("indptr / indices / data sizes disagree")
        if self.indices.size and (self.indices.min() < 0 or self.indices.max() >= n):
            raise IndexError("column index out of range")
        for i in range(m):
            c = self.indices[self.indptr[i]:self.indptr[i + 1]]
            if np.any(np.diff(c) <= 0):
                raise ValueError("columns of a row must be strictly increasing (no duplicates)")

    @property
    def nnz(self):
        return int(self.indices.size)

    def entries(self, I, J):
        """A[I][:, J] as float64 by the definition: row i is zero except data at indices."""
        I = np.asarray(I, np.int64)
        J = np.asarray(J, np.int64)
        out = np.zeros((I.size, J.size))
        for a, i in enumerate(I):
            row = np.zeros(self.shape[1])
            lo, hi = self.indptr[i], self.indptr[i + 1]
            row[self.indices[lo:hi]] = self.data[lo:hi]
            out[a] = row[J]
        return out

    def dense(self):
        return self.entries(np.arange(self.shape[0]), np.arange(self.shape[1]))


def _block(A, I, J):
    """A[I][:, J] as float64 for a dense array or an implicit / sparse source."""
    if isinstance(A, (RbfSource, CsrSource)):
        return A.entries(I, J)
    return np.asarray(A[np.ix_(I, J)], dtype=np.float64)


def gather(A, I, J):
    """P:195 "C = A_[:,I^c], R = A_[I^r,:], W = A_[I^r,I^c]".  Exact copies, as float64.
    A: dense array, or an implicit source whose entries are generated on access."""
    m, n = A.shape
    I = check_indices(I, m, "row index")
    J = check_indices(J, n, "column index")
    C = _block(A, np.arange(m), J)
    R = _block(A, I, np.arange(n))
    W = _block(A, I, J)
    return C, R, W


# --------------------------------------------------------------------------
# The k x k SVD of W ("Assuming an SVD W = U_w Sigma_w V_w^T")
# --------------------------------------------------------------------------
def canonical_signs(Uw, Vw):
    """Z5: flip each singular pair so the largest-|.| entry of U_w's column is
    positive (ties -> lowest row index).  Used so factor comparisons are direct;
    every product the method forms is invariant to it."""
    Uw = Uw.copy()
    Vw = Vw.copy()
    for i in range(Uw.shape[1]):
        col = Uw[:, i]
        if not np.any(col):
            continue
        p = int(np.argmax(np.abs(col)))  # first max -> lowest index
        if col[p] < 0:
            Uw[:, i] = -Uw[:, i]
            Vw[:, i] = -Vw[:, i]
    return Uw, Vw


def svd_w(W, tol=DEFAULT_TOL):
    """Thin SVD of W with sigma descending, truncated to sigma_i > tol*sigma_1 (Z4).

    Returns (Uw[k, r], sigma[r], Vw[k, r]).  LAPACK is used as a library step; it
    is pinned against closed forms in tests/test_oracle_sketch.py.
    """
    W = np.asarray(W, dtype=np.float64)
    if not np.all(np.isfinite(W)):
        raise ValueError("non-finite W")
    if W.size == 0:
        k = W.shape[0]
        return np.zeros((k, 0)), np.zeros(0), np.zeros((W.shape[1], 0))
    Uw, sig, Vwt = np.linalg.svd(W, full_matrices=False)
    Vw = Vwt.T
    if sig.size == 0 or sig[0] == 0.0:
        r = 0
    else:
        r = int(np.sum(sig > tol * sig[0]))
    Uw, Vw = canonical_signs(Uw[:, :r], Vw[:, :r])
    return Uw, sig[:r].copy(), Vw


# --------------------------------------------------------------------------
# The sketching routine and the pseudo-skeleton (Eq. 2)
# --------------------------------------------------------------------------
@dataclass
class Sketch:
    U: np.ndarray      # m x r, columns normalised ("U = C V_w N_c^-1")
    s: np.ndarray      # r, positive
    V: np.ndarray      # n x r ("V = N_r^-1 U_w^T R", stored as its transpose)
    sigma: np.ndarray  # singular values of W that survived (r,)
    Uw: np.ndarray
    Vw: np.ndarray
    Nc: np.ndarray
    Nr: np.ndarray

    @property
    def r(self):
        return self.s.size

    def dense(self):
        return (self.U * self.s) @ self.V.T


def sketch(C, R, W, m, n, k, mode=STABILIZED, tol=DEFAULT_TOL):
    """The paper's `sketching` routine, step by step.

    1. W = U_w Sigma_w V_w^T
    2. keep sigma_i > tol*sigma_1                              (Z4)
    3. extrapolate: Y_c = C V_w, Y_r = R^T U_w; N_c, N_r = column 2-norms
    4. drop components with a zero extrapolated norm           (Z4)
    5. U = Y_c N_c^-1, V = Y_r N_r^-1
    6. STABILIZED: s = sigma * sqrt(m n) / k                   (Z3)
       PSEUDO_SKELETON: s = N_c N_r / sigma, so U diag(s) V^T = C W_r^+ R exactly (Eq. 2)
    Order = sigma order; signs canonical (Z5).
    """
    C = np.asarray(C, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    Uw, sig, Vw = svd_w(W, tol)
    Yc = C @ Vw            # m x r
    Yr = R.T @ Uw          # n x r
    Nc = np.sqrt(np.sum(Yc * Yc, axis=0))
    Nr = np.sqrt(np.sum(Yr * Yr, axis=0))
    keep = (Nc > 0) & (Nr > 0)
    U = Yc[:, keep] / Nc[keep]
    V = Yr[:, keep] / Nr[keep]
    if mode == STABILIZED:
        s = sig[keep] * math.sqrt(float(m) * float(n)) / float(k)
    elif mode == PSEUDO_SKELETON:
        s = Nc[keep] * Nr[keep] / sig[keep]
    else:
        raise ValueError("unknown mode")
    return Sketch(U=U, s=s, V=V, sigma=sig[keep], Uw=Uw[:, keep], Vw=Vw[:, keep],
                  Nc=Nc[keep], Nr=Nr[keep])


def pseudo_skeleton_dense(C, R, W, tol=DEFAULT_TOL):
    """Eq. 2 written out: C W^+ R with the truncated pseudo-inverse (independent check)."""
    Uw, sig, Vw = svd_w(W, tol)
    Wp = (Vw / sig) @ Uw.T if sig.size else np.zeros((W.shape[1], W.shape[0]))
    return np.asarray(C, np.float64) @ Wp @ np.asarray(R, np.float64)


def embeddings(sk: Sketch):
    """Alg. 2 step 2: P = U S^1/2, Q = V S^1/2."""
    rs = np.sqrt(sk.s)
    return sk.U * rs, sk.V * rs


# --------------------------------------------------------------------------
# Weighted k-means (Eq. 6) with Lloyd iterations
# --------------------------------------------------------------------------
def weights(X, kind=WEIGHT_CONST, p=2.0):
    """w_l = Upsilon(||X_l||_2) (Eq. 6); constant for dense matrices (Z10)."""
    X = np.asarray(X, dtype=np.float64)
    if kind == WEIGHT_CONST:
        return np.ones(X.shape[0])
    if kind == WEIGHT_POWER:
        return np.sqrt(np.sum(X * X, axis=1)) ** p
    raise ValueError("unknown weight kind")


def sq_dist(X, c):
    """||X_l - c||^2 for every row l, by direct differences (Z18 / F3)."""
    D = np.asarray(X, np.float64) - np.asarray(c, np.float64)[None, :]
    return np.sum(D * D, axis=1)


def sq_dist_all(X, centres, chunk=4096):
    """N x k2 matrix of direct-difference squared distances."""
    X = np.asarray(X, np.float64)
    centres = np.asarray(centres, np.float64)
    out = np.empty((X.shape[0], centres.shape[0]))
    for a in range(0, X.shape[0], chunk):
        Xb = X[a:a + chunk]
        D = Xb[:, None, :] - centres[None, :, :]
        out[a:a + chunk] = np.sum(D * D, axis=2)
    return out


def argmin_with_gap(Dm):
    """Lowest-index argmin per row (Z11) and relative gap (d2 - d1)/d2 (Z18)."""
    lab = np.argmin(Dm, axis=1)
    d1 = Dm[np.arange(Dm.shape[0]), lab]
    if Dm.shape[1] > 1:
        part = np.partition(Dm, 1, axis=1)
        d2 = part[:, 1]
        with np.errstate(invalid="ignore", divide="ignore"):
            gap = np.where(d2 > 0, (d2 - d1) / d2, 0.0)
    else:
        gap = np.full(Dm.shape[0], np.inf)
    return lab.astype(np.int64), d1, gap


@dataclass
class KmeansResult:
    centres: np.ndarray          # k2 x d after the c-th update
    labels: np.ndarray           # assignment of the c-th iteration
    objective: np.ndarray        # J_t, t = 1..c (Eq. 6 at the t-th assignment)
    cluster_w: np.ndarray        # omega_j from the c-th assignment
    gaps: list = field(default_factory=list)       # per-iteration relative gaps
    labels_hist: list = field(default_factory=list)
    centres_hist: list = field(default_factory=list)  # centres used by iteration t


def lloyd(X, k2, iters, w=None, init_idx=None, init_centres=None, seed=0,
          tag=rng.TAG_INIT_ROWS, check_monotone=True):
    """Weighted Lloyd iterations (O6; Eq. 6; c iterations P:204).

    init: centres = X[Floyd(N, k2, tag)] (Z9), or explicit indices / centres.
    each iteration t: s_t(l) = argmin_j ||X_l - c_j||^2 (direct differences,
    lowest j on ties); J_t = sum_l w_l ||X_l - c_{s_t(l)}||^2; then every cluster
    with positive weight moves to its weighted mean, others keep their centre (Z12).
    """
    X = np.asarray(X, np.float64)
    N = X.shape[0]
    if w is None:
        w = np.ones(N)
    w = np.asarray(w, np.float64)
    if k2 < 1 or iters < 1:
        raise ValueError("k2 >= 1 and iters >= 1 required")
    if int(np.sum(w > 0)) < k2:
        raise ValueError("fewer than k2 points with nonzero weight")
    if init_centres is not None:
        centres = np.array(init_centres, dtype=np.float64, copy=True)
    else:
        if init_idx is None:
            init_idx = rng.floyd(N, k2, seed, tag)
        centres = X[np.asarray(init_idx, dtype=np.int64)].copy()
    res = KmeansResult(centres=None, labels=None, objective=np.zeros(iters), cluster_w=None)
    for t in range(iters):
        res.centres_hist.append(centres.copy())
        Dm = sq_dist_all(X, centres)
        lab, d1, gap = argmin_with_gap(Dm)
        res.objective[t] = float(np.sum(w * d1))
        res.gaps.append(gap)
        res.labels_hist.append(lab)
        cw = np.bincount(lab, weights=w, minlength=k2)
        new = centres.copy()
        for j in range(k2):
            if cw[j] > 0:
                sel = lab == j
                new[j] = np.sum(w[sel, None] * X[sel], axis=0) / cw[j]
        centres = new
        res.labels = lab
        res.cluster_w = cw
    if check_monotone:
        # P8: J_{t+1} <= J_t up to rounding; the slack is relative to the data scale
        # sum_l w_l ||X_l||^2 so exact-zero objectives tolerate the rounding of a mean.
        ob = res.objective
        scale = float(np.sum(w * np.sum(X * X, axis=1)))
        for t in range(1, iters):
            if ob[t] > ob[t - 1] + 1e-12 * (ob[t - 1] + scale):
                raise AssertionError(f"Lloyd objective increased at t={t}: {ob[t-1]} -> {ob[t]}")
    res.centres = centres
    return res


def encoding_error(X, reps, assignment, w=None):
    """Eq. 3 / Eq. 6: sum_l w_l ||X_l - X_{reps[s(l)]}||^2."""
    X = np.asarray(X, np.float64)
    if w is None:
        w = np.ones(X.shape[0])
    Z = X[np.asarray(reps, dtype=np.int64)][np.asarray(assignment, dtype=np.int64)]
    return float(np.sum(np.asarray(w) * np.sum((X - Z) ** 2, axis=1)))


@dataclass
class SnapResult:
    reps_sorted: np.ndarray   # the follow-up index set, ascending
    rep_of_centre: np.ndarray  # representative chosen by centre j
    gap: np.ndarray           # relative gap best vs runner-up untaken point, per centre
    order: np.ndarray         # visiting order of centres


def snap(X, centres, cluster_w):
    """P:169 "any k-means clustering center will be replaced with its closest
    in-sample point"; duplicates resolved greedily in order (-omega_j, j), each
    centre taking its nearest untaken point, lowest index on ties (Z13)."""
    X = np.asarray(X, np.float64)
    k2 = centres.shape[0]
    order = sorted(range(k2), key=lambda j: (-float(cluster_w[j]), j))
    taken = np.zeros(X.shape[0], dtype=bool)
    rep = np.full(k2, -1, dtype=np.int64)
    gap = np.zeros(k2)
    for j in order:
        d = sq_dist(X, centres[j])
        d = np.where(taken, np.inf, d)
        l = int(np.argmin(d))
        if not np.isfinite(d[l]):
            raise ValueError("no untaken point left for centre")
        d1 = d[l]
        d[l] = np.inf
        d2 = float(np.min(d)) if d.size > 1 else np.inf
        gap[j] = (d2 - d1) / d2 if (np.isfinite(d2) and d2 > 0) else (0.0 if d2 == 0 else np.inf)
        rep[j] = l
        taken[l] = True
    return SnapResult(reps_sorted=np.sort(rep), rep_of_centre=rep, gap=gap,
                      order=np.array(order, dtype=np.int64))


# --------------------------------------------------------------------------
# Hard-threshold follow-up (P:312 variant (f))
# --------------------------------------------------------------------------
def row_sq_norms(X):
    """||X_l||^2 per row, accumulated in float64 over the columns IN ORDER (Z26: the
    ranking key of the hard threshold; with float32 inputs every square is exact in
    float64, so the value is fixed by this summation order)."""
    X = np.asarray(X, np.float64)
    acc = np.zeros(X.shape[0])
    for i in range(X.shape[1]):
        acc = acc + X[:, i] * X[:, i]
    return acc


def hard_threshold_select(w, k):
    """P:312 (f) "top-k samples with largest weighting coefficients (Eq. 6)", S:182-186:
    the indices of the k largest w_l, ties to the lowest index, returned ascending."""
    w = np.asarray(w, np.float64)
    if not (1 <= k <= w.shape[0]):
        raise ValueError("need 1 <= k <= len(w)")
    order = sorted(range(w.shape[0]), key=lambda l: (-float(w[l]), l))
    return np.sort(np.array(order[:k], dtype=np.int64))


def hard_threshold_followup(X, k):
    """Follow-up indices of variant (f) on an embedding X: the weighting coefficient
    Upsilon(||X_l||) is monotone in ||X_l|| (Eq. 6; power Upsilon, p > 0), so its top-k is
    the top-k of ||X_l||^2 (Z26)."""
    return hard_threshold_select(row_sq_norms(X), k)


# --------------------------------------------------------------------------
# Orthogonalization (Supp. section 3) and the leverage-score follow-up
# (P:312 variant (e))
# --------------------------------------------------------------------------
def orthogonalize(U, s, V):
    """Supp. section 3, step by step: U = U0 S0 V0^T (thin SVD); then
    S0 V0^T diag(s) V^T = U1 S1 V1^T; the result is (U0 U1, S1, V1), i.e. A ~ (U0 U1) S1 V1^T.
    Components with S1 <= tol * S1_max (Z4's rule) are dropped (a rank-deficient input)."""
    U = np.asarray(U, np.float64)
    V = np.asarray(V, np.float64)
    s = np.asarray(s, np.float64)
    U0, S0, V0t = np.linalg.svd(U, full_matrices=False)
    B = (S0[:, None] * V0t) @ (s[:, None] * V.T)
    U1, S1, V1t = np.linalg.svd(B, full_matrices=False)
    keep = S1 > DEFAULT_TOL * S1[0] if S1.size and S1[0] > 0 else np.zeros(S1.size, dtype=bool)
    return U0 @ U1[:, keep], S1[keep], V1t[keep].T


def leverage_scores(F):
    """Approximate leverage scores l_i = ||F_i||^2 / r of a factor with orthonormal columns
    (P:312 (e)); r = number of columns.  ||F_i||^2 as in row_sq_norms."""
    F = np.asarray(F, np.float64)
    return row_sq_norms(F) / F.shape[1]


def leverage_sample(F, k, seed, tag):
    """k distinct indices drawn without replacement with probability proportional to the
    leverage scores, as Efraimidis-Spirakis keys: point l gets the key
    l_l / (-log u_l) with u_l = rng.uniform01(seed, tag, l) (the ranking of u^(1/l_l)); the k
    largest keys win (ties -> lowest index), returned ascending (Z27)."""
    w = leverage_scores(F)
    if not (1 <= k <= int(np.count_nonzero(w))):
        raise ValueError("need 1 <= k <= number of nonzero leverage scores")
    u = rng.uniform01(seed, tag, np.arange(w.shape[0]))
    return hard_threshold_select(w / -np.log(u), k)


# --------------------------------------------------------------------------
# Residual  ||A - U diag(s) V^T||_F -- the evaluation step
# --------------------------------------------------------------------------
def residual(A, F, G, s=None, block=2048):
    """Returns (r^2, a^2) with r^2 = sum_ij (A - F diag(s) G^T)_ij^2, a^2 = sum A^2,
    accumulated in float64 over row blocks (O9)."""
    F = np.asarray(F, np.float64)
    G = np.asarray(G, np.float64)
    if s is not None:
        F = F * np.asarray(s, np.float64)[None, :]
    r2 = 0.0
    a2 = 0.0
    n = A.shape[1]
    for i in range(0, A.shape[0], block):
        Ab = _block(A, np.arange(i, min(i + block, A.shape[0])), np.arange(n))
        E = Ab - F[i:i + block] @ G.T
        r2 += float(np.sum(E * E))
        a2 += float(np.sum(Ab * Ab))
    return r2, a2


def residual_sparse(A, F, G, s=None):
    """The P:313 error of a sparse A (CsrSource) without forming A - F diag(s) G^T:
        ||A - B||_F^2 = ||A||_F^2 - 2 <A, B> + ||B||_F^2,   B = F S G^T, S = diag(s),
    where <A, B> = sum over the nonzeros a_ij of a_ij (F S G^T)_ij and
        ||B||_F^2 = trace(S F^T F S G^T G) = sum_kl (F^T F)_kl s_k s_l (G^T G)_kl
    (the r x r Gram products).  Returns (r^2, a^2) like residual()."""
    F = np.asarray(F, np.float64)
    G = np.asarray(G, np.float64)
    sv = np.ones(F.shape[1]) if s is None else np.asarray(s, np.float64)
    a2 = float(np.sum(A.data * A.data))
    cross = 0.0
    for i in range(A.shape[0]):
        lo, hi = A.indptr[i], A.indptr[i + 1]
        if hi > lo:
            b = G[A.indices[lo:hi]] @ (F[i] * sv)     # (F S G^T)_ij at the row's nonzero columns
            cross += float(np.sum(A.data[lo:hi] * b))
    gf = F.T @ F
    gg = G.T @ G
    b2 = float(np.sum(gf * np.outer(sv, sv) * gg))
    return a2 - 2.0 * cross + b2, a2


def residual_sampled(A, F, G, i, j, s=None, chunk=1 << 20, f_rows=None):
    """The P:313 error on a uniform subset of entries (BASELINE.json configs[4] "residual
    estimated on a seeded 1e9-entry uniform subset"; reading Z23: T i.i.d. positions (i_t, j_t)).
    Unbiased estimates of sum (A - F diag(s) G^T)^2 and sum A^2:
        r2 = (m n / T) sum_t (A_{i_t j_t} - F_{i_t} . G_{j_t})^2,   a2 = (m n / T) sum_t A_{i_t j_t}^2.
    f_rows: optional int array, F's row of pair t is F[f_rows[t]] (F given as the rows i_t only)."""
    m, n = A.shape
    i = np.asarray(i, np.int64)
    j = np.asarray(j, np.int64)
    T = i.shape[0]
    F = np.asarray(F, np.float64)
    G = np.asarray(G, np.float64)
    if s is not None:
        F = F * np.asarray(s, np.float64)[None, :]
    r2 = 0.0
    a2 = 0.0
    for c in range(0, T, chunk):
        ic, jc = i[c:c + chunk], j[c:c + chunk]
        fc = ic if f_rows is None else np.asarray(f_rows, np.int64)[c:c + chunk]
        if isinstance(A, RbfSource):
            a = A.at(ic, jc)
        elif isinstance(A, CsrSource):
            a = np.array([A.entries([x], [y])[0, 0] for x, y in zip(ic, jc)])
        else:
            a = np.asarray(A[ic, jc], np.float64)
        e = a - np.sum(F[fc] * G[jc], axis=1)
        r2 += float(np.sum(e * e))
        a2 += float(np.sum(a * a))
    scale = float(m) * float(n) / float(T)
    return scale * r2, scale * a2


def relative_error(A, F, G, s=None):
    r2, a2 = residual(A, F, G, s)
    if a2 == 0.0:
        raise ZeroDivisionError("||A||_F = 0: relative error undefined")
    return math.sqrt(r2 / a2)


# --------------------------------------------------------------------------
# Algorithm 2 end to end
# --------------------------------------------------------------------------
@dataclass
class CabsResult:
    I: np.ndarray
    J: np.ndarray
    pilot: Sketch
    P: np.ndarray
    Q: np.ndarray
    km_rows: KmeansResult
    km_cols: KmeansResult
    snap_rows: SnapResult
    snap_cols: SnapResult
    Ibar: np.ndarray
    Jbar: np.ndarray
    follow: Sketch
    resid_sq: float = float("nan")
    a_sq: float = float("nan")


def cabs_run(A, k1, k2, iters, seed=0, mode=STABILIZED, tol=DEFAULT_TOL,
             weight_kind=WEIGHT_CONST, weight_p=2.0, I=None, J=None,
             init_rows=None, init_cols=None, with_residual=True, followup="kmeans", n_samples=0):
    """Algorithm 2 plus the evaluation residual.  followup="hard" /
    "leverage" replaces step 3 by the paper's variant (f) / (e) of P:312 (km_* / snap_* are None).
    A: dense array, RbfSource or CsrSource.  n_samples > 0: the residual is the sampled estimate on the
    pairs rng.residual_pairs(seed, n_samples, m, n)."""
    m, n = A.shape
    if not (1 <= k1 <= min(m, n)) or not (1 <= k2 <= min(m, n)):
        raise ValueError("need 1 <= k1, k2 <= min(m, n)")
    # step 1: pilot sampling
    if I is None:
        I = rng.floyd(m, k1, seed, rng.TAG_PILOT_ROWS)
    if J is None:
        J = rng.floyd(n, k1, seed, rng.TAG_PILOT_COLS)
    C, R, W = gather(A, I, J)
    # step 2: pilot sketching, P = U S^1/2, Q = V S^1/2
    pilot = sketch(C, R, W, m, n, k1, mode, tol)
    P, Q = embeddings(pilot)
    if followup == "hard":  # P:312 (f): top-k2 weighting coefficients on each side
        Ib, Jb = hard_threshold_followup(P, k2), hard_threshold_followup(Q, k2)
        Cb, Rb, Wb = gather(A, Ib, Jb)
        follow = sketch(Cb, Rb, Wb, m, n, k2, mode, tol)
        res = CabsResult(I=I, J=J, pilot=pilot, P=P, Q=Q, km_rows=None, km_cols=None,
                         snap_rows=None, snap_cols=None, Ibar=Ib, Jbar=Jb, follow=follow)
        if with_residual:
            res.resid_sq, res.a_sq = _evaluate(A, follow, seed, n_samples)
        return res
    if followup == "leverage":  # P:312 (e): orthogonalize the pilot (Supp. 3), sample by leverage
        Uo, so, Vo = orthogonalize(pilot.U, pilot.s, pilot.V)
        Ib = leverage_sample(Uo, k2, seed, rng.TAG_LEVERAGE_ROWS)
        Jb = leverage_sample(Vo, k2, seed, rng.TAG_LEVERAGE_COLS)
        Cb, Rb, Wb = gather(A, Ib, Jb)
        follow = sketch(Cb, Rb, Wb, m, n, k2, mode, tol)
        res = CabsResult(I=I, J=J, pilot=pilot, P=P, Q=Q, km_rows=None, km_cols=None,
                         snap_rows=None, snap_cols=None, Ibar=Ib, Jbar=Jb, follow=follow)
        if with_residual:
            res.resid_sq, res.a_sq = _evaluate(A, follow, seed, n_samples)
        return res
    if followup != "kmeans":
        raise ValueError("followup must be 'kmeans', 'hard' or 'leverage'")
    # step 3: weighted k-means on P and Q, snap to in-sample points
    km_r = lloyd(P, k2, iters, weights(P, weight_kind, weight_p), init_idx=init_rows,
                 seed=seed, tag=rng.TAG_INIT_ROWS)
    km_c = lloyd(Q, k2, iters, weights(Q, weight_kind, weight_p), init_idx=init_cols,
                 seed=seed, tag=rng.TAG_INIT_COLS)
    sn_r = snap(P, km_r.centres, km_r.cluster_w)
    sn_c = snap(Q, km_c.centres, km_c.cluster_w)
    Ib, Jb = sn_r.reps_sorted, sn_c.reps_sorted
    # step 4: follow-up sketching
    Cb, Rb, Wb = gather(A, Ib, Jb)
    follow = sketch(Cb, Rb, Wb, m, n, k2, mode, tol)
    res = CabsResult(I=I, J=J, pilot=pilot, P=P, Q=Q, km_rows=km_r, km_cols=km_c,
                     snap_rows=sn_r, snap_cols=sn_c, Ibar=Ib, Jbar=Jb, follow=follow)
    if with_residual:
        res.resid_sq, res.a_sq = _evaluate(A, follow, seed, n_samples)
    return res


# --------------------------------------------------------------------------
# the baselines of Section 2.2 on the same gathers -- BR-CUR (Algorithm 1,
# P:83-103), Sketch-CUR (target rate 3x the base rate P:312 (a)) -- and the rank sweep
# on a validation set ("use a validation set to choose the optimal number of
# singular vectors")
# --------------------------------------------------------------------------
def pinv(X, tol=DEFAULT_TOL):
    """Moore-Penrose pseudo-inverse by the thin SVD, singular values <= tol * sigma_1 dropped
    (the truncation rule of the sketching routine)."""
    X = np.asarray(X, np.float64)
    U, sig, Vt = np.linalg.svd(X, full_matrices=False)
    if sig.size == 0 or sig[0] == 0.0:
        return np.zeros(X.T.shape)
    r = int(np.sum(sig > tol * sig[0]))
    return (Vt[:r].T / sig[:r]) @ U[:, :r].T


@dataclass
class CurResult:
    C: np.ndarray   # m x k1 = A[:, base cols]
    U: np.ndarray   # k1 x k1 middle matrix U*
    R: np.ndarray   # k1 x n = A[base rows, :]

    def dense(self):
        return self.C @ self.U @ self.R


def br_cur(A, Ibr, Ibc, Itr, Itc, tol=DEFAULT_TOL):
    """Algorithm 1 step by step: 1 C = A[:, I^b_c], R = A[I^b_r, :]; 2 C_bar =
    C[I^t_r, :], R_bar = R[:, I^t_c]; 3 M = A[I^t_r, I^t_c]; 4 U* = argmin ||M - C_bar U R_bar||_F
    = C_bar^+ M R_bar^+ (the minimum-norm least-squares solution); 5 A ~ C U* R."""
    m, n = A.shape
    Ibr, Ibc = check_indices(Ibr, m, "base row"), check_indices(Ibc, n, "base column")
    Itr, Itc = check_indices(Itr, m, "target row"), check_indices(Itc, n, "target column")
    if Itr.size == 0 or Itc.size == 0:
        raise ValueError("empty target sampling: M undefined")
    C = _block(A, np.arange(m), Ibc)
    R = _block(A, Ibr, np.arange(n))
    Cb = C[Itr, :]
    Rb = R[:, Itc]
    M = _block(A, Itr, Itc)
    U = pinv(Cb, tol) @ M @ pinv(Rb, tol)
    return CurResult(C=C, U=U, R=R)


def sketch_cur(A, Ibr, Ibc, mult, seed, tol=DEFAULT_TOL):
    """Sketch-CUR: BR-CUR with target rows / columns drawn uniformly and
    independently of the base sampling (Floyd, tags TAG_TARGET_ROWS / _COLS), mult times as many
    (P:312 (a): "the target sampling rate is chosen three times as much as the base")."""
    m, n = A.shape
    kt = mult * len(Ibr)
    if kt > min(m, n):
        raise ValueError("target sample larger than the matrix")
    Itr = rng.floyd(m, kt, seed, rng.TAG_TARGET_ROWS)
    Itc = rng.floyd(n, kt, seed, rng.TAG_TARGET_COLS)
    return br_cur(A, Ibr, Ibc, Itr, Itc, tol), Itr, Itc


def holdout_indices(N, h, seed, tag, exclude):
    """A validation sample: h uniform indices (Floyd, tag) less those in `exclude`
    (the sketch's own rows or columns), ascending."""
    idx = rng.floyd(N, h, seed, tag)
    return idx[~np.isin(idx, np.asarray(exclude, np.int64))]


def holdout_errors(A, U, s, V, Hr, Hc):
    """The rank sweep on the validation block ("approximation error varies with the
    number of singular vectors used"): e[rho] = ||A[Hr, Hc] - U[Hr, :rho] diag(s[:rho])
    V[Hc, :rho]^T||_F^2 for rho = 0 .. r, by the definition (FP64)."""
    B = _block(A, np.asarray(Hr, np.int64), np.asarray(Hc, np.int64))
    Uh = np.asarray(U, np.float64)[np.asarray(Hr, np.int64)]
    Vh = np.asarray(V, np.float64)[np.asarray(Hc, np.int64)]
    sv = np.asarray(s, np.float64)
    r = sv.size
    return np.array([float(np.sum((B - (Uh[:, :rho] * sv[:rho]) @ Vh[:, :rho].T) ** 2)) for rho in range(r + 1)])


def validate_rank(errors):
    """the rank rho in 1..r with the smallest validation error, lowest on ties."""
    e = np.asarray(errors, np.float64)
    if e.size < 2:
        raise ValueError("empty sweep")
    return int(np.argmin(e[1:])) + 1


def _evaluate(A, follow, seed, n_samples):
    if n_samples > 0:
        m, n = A.shape
        i, j = rng.residual_pairs(seed, n_samples, m, n)
        return residual_sampled(A, follow.U, follow.V, i, j, follow.s)
    return residual(A, follow.U, follow.V, follow.s)
