"""Pins for the oracle's hard-threshold follow-up (P:312 variant (f)).

Golden examples of S:188-189, brute force over all C(n, k) subsets, closed-form
squared norms, the monotone-Upsilon equivalence (Z26), and an end-to-end exactness case
(pseudo-skeleton reconstruction of an exact low-rank matrix from the selected rows and
columns).
"""
import itertools
import os

import numpy as np
import pytest

from oracle import cabs as O
from oracle import rng


def _golden(golden_dir):
    cases = []
    with open(os.path.join(golden_dir, "hard_threshold_S188.txt")) as f:
        for line in f:
            if not line.startswith("case"):
                continue
            lhs, rhs = line.split("->")
            vals = lhs.split()[1:]
            cases.append((int(vals[0]), [float(v) for v in vals[1:]], [int(v) for v in rhs.split()]))
    return cases


def test_golden_examples(golden_dir):
    cases = _golden(golden_dir)
    assert len(cases) == 2
    for k, w, want in cases:
        assert O.hard_threshold_select(np.array(w), k).tolist() == want


@pytest.mark.parametrize("seed", range(12))
def test_brute_force_subsets(seed):
    g = np.random.default_rng(seed)
    n = int(g.integers(1, 11))
    k = int(g.integers(1, n + 1))
    w = g.integers(0, 5, size=n).astype(np.float64)  # small integers: many ties
    best = None
    for sub in itertools.combinations(range(n), k):  # lexicographic order
        sm = w[list(sub)].sum()
        if best is None or sm > best[0]:
            best = (sm, sub)
    assert O.hard_threshold_select(w, k).tolist() == list(best[1])


def test_bad_k():
    with pytest.raises(ValueError):
        O.hard_threshold_select(np.ones(3), 0)
    with pytest.raises(ValueError):
        O.hard_threshold_select(np.ones(3), 4)


def test_row_sq_norms_closed_form():
    X = np.array([[3.0, 4.0, 0.0], [1.0, 2.0, 2.0], [0.0, 0.0, 0.0], [-2.0, 0.5, 0.25]], dtype=np.float32)
    assert O.row_sq_norms(X).tolist() == [25.0, 9.0, 0.0, 4.3125]
    g = np.random.default_rng(3)
    Y = g.standard_normal((50, 7)).astype(np.float32)
    assert np.array_equal(O.row_sq_norms(2 * Y), 4 * O.row_sq_norms(Y))  # powers of two are exact
    assert np.allclose(O.row_sq_norms(Y), np.linalg.norm(Y.astype(np.float64), axis=1) ** 2, rtol=1e-14)


@pytest.mark.parametrize("p", [0.5, 1.0, 2.0, 3.0])
def test_monotone_upsilon_equivalence(p):
    """Z26: the top-k of Upsilon(||X_l||) for the power Upsilon (Eq. 6) is the top-k of ||X_l||^2."""
    g = np.random.default_rng(int(10 * p))
    X = g.standard_normal((300, 9))
    for k in (1, 17, 300):
        want = O.hard_threshold_select(O.weights(X, O.WEIGHT_POWER, p), k)
        assert O.hard_threshold_followup(X, k).tolist() == want.tolist()


def test_followup_exact_low_rank():
    """Variant (f) end to end: A of exact rank 4 with a few heavy rows / columns; the
    hard threshold picks the heaviest embedding rows, and the pseudo-skeleton on those
    k2 >= rank rows and columns reconstructs A to rounding (Eq. 2)."""
    g = np.random.default_rng(7)
    m, n, r, k = 60, 45, 4, 8
    F = g.standard_normal((m, r)); G = g.standard_normal((n, r))
    F[[3, 17, 40]] *= 20.0
    G[[5, 30]] *= 15.0
    A = F @ G.T
    res = O.cabs_run(A, 10, k, 5, seed=1, mode=O.PSEUDO_SKELETON, followup="hard")
    assert res.km_rows is None and res.snap_rows is None
    assert res.Ibar.tolist() == O.hard_threshold_select(O.row_sq_norms(res.P), k).tolist()
    assert {3, 17, 40} <= set(res.Ibar.tolist())
    assert {5, 30} <= set(res.Jbar.tolist())
    assert np.sqrt(res.resid_sq / res.a_sq) < 1e-9
    with pytest.raises(ValueError):
        O.cabs_run(A, 10, k, 5, followup="nope")
