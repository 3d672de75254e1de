"""Pins for the oracle's weighted Lloyd k-means and snap (oracle/cabs.py).

P7 (brute force on <= 12 points; S:163 golden example), P8 (Lloyd
monotonicity), P9 (encoding error), snap rules Z11-Z14.
"""
import itertools
import os

import numpy as np
import pytest

from oracle import cabs as O


def _golden_1d(golden_dir):
    d = {}
    with open(os.path.join(golden_dir, "kmeans_1d_S163.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            key, *vals = line.split()
            d[key] = [float(v) for v in vals]
    return d


def _brute_force_opt(X, k, w):
    """Global optimum of Eq. 6 over all k^N labelings (each label set -> weighted means)."""
    best = np.inf
    N = X.shape[0]
    for lab in itertools.product(range(k), repeat=N):
        lab = np.array(lab)
        obj = 0.0
        for j in range(k):
            sel = lab == j
            if not np.any(sel) or w[sel].sum() == 0:
                continue
            c = np.sum(w[sel, None] * X[sel], axis=0) / w[sel].sum()
            obj += float(np.sum(w[sel] * np.sum((X[sel] - c) ** 2, axis=1)))
        best = min(best, obj)
    return best


def test_golden_1d_example(golden_dir):
    g = _golden_1d(golden_dir)
    X = np.array(g["points"])[:, None]
    for init in ([0, 1], [3, 4], [0, 4], [1, 2]):
        km = O.lloyd(X, int(g["k"][0]), 10, init_idx=init)
        assert np.allclose(np.sort(km.centres[:, 0]), g["centres"])
        lab = km.labels
        part = (lab == lab[4]).astype(int)                  # cluster of point 11 -> 1
        assert part.tolist() == [int(v) for v in g["partition"]]
        assert abs(km.objective[-1] - g["objective"][0]) < 1e-12
        sn = O.snap(X, km.centres, km.cluster_w)
        assert sn.reps_sorted.tolist() == [int(v) for v in g["representatives"]]
        j = int(np.argmax(km.centres[:, 0]))               # centre 10.5: exact tie 10 vs 11
        assert sn.gap[j] == 0.0 and sn.rep_of_centre[j] == 3


@pytest.mark.parametrize("seed", range(8))
def test_brute_force_optimum_well_separated(seed):
    g = np.random.default_rng(seed)
    k = 3
    means = np.array([[0.0, 0.0], [10.0, 0.0], [0.0, 10.0]])
    N = 9
    lab = np.repeat(np.arange(k), 3)
    X = means[lab] + 0.3 * g.standard_normal((N, 2))
    w = np.ones(N)
    init = [int(np.where(lab == j)[0][0]) for j in range(k)]
    km = O.lloyd(X, k, 10, w, init_idx=init)
    assert abs(km.objective[-1] - _brute_force_opt(X, k, w)) < 1e-9


@pytest.mark.parametrize("seed", range(6))
def test_lloyd_output_is_fixed_point(seed):
    g = np.random.default_rng(100 + seed)
    N, k = 8, 3
    X = g.standard_normal((N, 2))
    w = g.uniform(0.5, 2.0, N)
    km = O.lloyd(X, k, 30, w, seed=seed)
    # nearest assignment w.r.t. the centres it used last, and the centres are weighted means
    last_c = km.centres_hist[-1]
    D = ((X[:, None, :] - last_c[None]) ** 2).sum(-1)
    assert np.array_equal(km.labels, np.argmin(D, axis=1))
    opt = _brute_force_opt(X, k, w)
    assert km.objective[-1] >= opt - 1e-9                   # never below the global optimum


def test_distinct_points_zero_objective():
    X = np.random.default_rng(0).standard_normal((5, 3))
    km = O.lloyd(X, 5, 3, init_idx=[0, 1, 2, 3, 4])
    assert km.objective[0] == 0.0 and km.objective[-1] == 0.0


def test_zero_weight_points_do_not_change_objective():
    g = np.random.default_rng(1)
    X = g.standard_normal((8, 2))
    w = np.ones(8)
    km1 = O.lloyd(X, 2, 5, w, init_idx=[0, 1])
    Xz = np.vstack([X, 50 + g.standard_normal((3, 2))])      # far-away zero-weight points
    wz = np.concatenate([w, np.zeros(3)])
    km2 = O.lloyd(Xz, 2, 5, wz, init_idx=[0, 1])
    assert np.allclose(km1.objective, km2.objective, rtol=1e-14)
    assert np.allclose(km1.centres, km2.centres)


def test_constant_weight_equals_unweighted():
    g = np.random.default_rng(2)
    X = g.standard_normal((40, 3))
    a = O.lloyd(X, 4, 6, None, seed=5)
    b = O.lloyd(X, 4, 6, O.weights(X, O.WEIGHT_CONST), seed=5)
    assert np.array_equal(a.labels, b.labels) and np.array_equal(a.centres, b.centres)


def test_power_weights():
    X = np.array([[3.0, 4.0], [0.0, 0.0]])
    assert O.weights(X, O.WEIGHT_POWER, 2.0).tolist() == [25.0, 0.0]
    assert O.weights(X, O.WEIGHT_CONST).tolist() == [1.0, 1.0]


@pytest.mark.parametrize("seed", range(10))
def test_lloyd_monotone(seed):
    g = np.random.default_rng(200 + seed)
    X = np.vstack([g.standard_normal((50, 4)) + 3 * g.standard_normal(4) for _ in range(5)])
    w = O.weights(X, O.WEIGHT_POWER, 2.0) if seed % 2 else None
    km = O.lloyd(X, 7, 15, w, seed=seed)         # asserts J_{t+1} <= J_t internally (P8)
    assert np.all(np.diff(km.objective) <= 1e-12 * km.objective[:-1])


def test_empty_cluster_keeps_centre():
    X = np.array([[0.0], [1.0], [2.0]])
    km = O.lloyd(X, 2, 2, init_centres=np.array([[1.0], [100.0]]))
    assert km.centres[1, 0] == 100.0 and km.cluster_w[1] == 0.0


def test_too_few_weighted_points():
    with pytest.raises(ValueError):
        O.lloyd(np.zeros((3, 2)), 2, 1, np.array([1.0, 0.0, 0.0]))


def test_encoding_error_examples():
    X = np.array([[0.0], [2.0]])
    assert O.encoding_error(X, [0, 1], [0, 1]) == 0.0
    assert O.encoding_error(X, [0], [0, 0]) == 4.0
    g = np.random.default_rng(3)                             # S:172 brute force
    Xr = g.standard_normal((6, 2))
    reps = [0, 3]
    near = np.argmin(((Xr[:, None] - Xr[reps][None]) ** 2).sum(-1), axis=1)
    e_near = O.encoding_error(Xr, reps, near)
    for a in itertools.product(range(2), repeat=6):
        assert e_near <= O.encoding_error(Xr, reps, a) + 1e-12


def test_snap_dedupe_greedy_by_weight():
    # two centres both nearest to point 0; heavier centre wins, lighter takes runner-up
    X = np.array([[0.0], [1.0], [5.0]])
    centres = np.array([[0.1], [0.0]])
    sn = O.snap(X, centres, np.array([1.0, 3.0]))
    assert sn.rep_of_centre.tolist() == [1, 0] and sn.reps_sorted.tolist() == [0, 1]
    sn = O.snap(X, centres, np.array([3.0, 1.0]))
    assert sn.rep_of_centre.tolist() == [0, 1]
    sn = O.snap(X, centres, np.array([2.0, 2.0]))            # equal weights -> lower centre first
    assert sn.rep_of_centre.tolist() == [0, 1]


def test_snap_over_all_points_not_members():
    # Z13: the snap searches all points, not only the centre's cluster members
    X = np.array([[0.0], [0.9], [2.0]])
    sn = O.snap(X, np.array([[1.0], [2.0]]), np.array([1.0, 1.0]))
    assert sn.rep_of_centre.tolist() == [1, 2]


def test_argmin_with_gap_closed_form():
    """The gap that decides which GPU/oracle label flips are excused (Z18): lowest-index argmin,
    relative gap (d2 - d1) / d2 to the runner-up, 0 for an exact tie, 0 when d2 = 0, inf with
    one centre; checked on distances with known values, and on points against centres at known
    positions (x = 0 against centres at 1 and 3 -> d = 1, 9 -> gap 8/9)."""
    D = np.array([[1.0, 4.0, 9.0],   # unique minimum: gap (4 - 1) / 4
                  [2.0, 2.0, 5.0],   # exact tie -> lowest index, gap 0
                  [7.0, 3.0, 3.5],   # minimum in the middle: gap (3.5 - 3) / 3.5
                  [0.0, 0.0, 1.0],   # d2 = 0 -> gap 0
                  [5.0, 0.0, 5.0]])  # zero distance, runner-up 5: gap 1
    lab, d1, gap = O.argmin_with_gap(D)
    assert lab.tolist() == [0, 0, 1, 0, 1]
    assert d1.tolist() == [1.0, 2.0, 3.0, 0.0, 0.0]
    assert np.allclose(gap, [0.75, 0.0, 0.5 / 3.5, 0.0, 1.0], rtol=0, atol=1e-15)
    lab1, _, gap1 = O.argmin_with_gap(np.array([[2.0], [0.5]]))
    assert lab1.tolist() == [0, 0] and np.all(np.isinf(gap1))
    X = np.array([[0.0], [2.0], [2.9]])
    cen = np.array([[1.0], [3.0]])
    lab2, d12, gap2 = O.argmin_with_gap(O.sq_dist_all(X, cen))
    assert lab2.tolist() == [0, 0, 1]  # x = 2 is equidistant: lowest index
    assert np.allclose(d12, [1.0, 1.0, 0.01], rtol=0, atol=1e-12)
    assert np.allclose(gap2, [8.0 / 9.0, 0.0, (3.61 - 0.01) / 3.61], rtol=0, atol=1e-12)
