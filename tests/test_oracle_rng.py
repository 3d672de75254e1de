"""Pins for the oracle's counter-based RNG (oracle/rng.py).

Philox is pinned to published known-answer vectors; Lemire to the counting
argument of its acceptance region; Floyd to SPEC's examples and to
exact uniformity over subsets.
"""
import math
import os

import numpy as np
import pytest

from oracle import rng


def _kat(golden_dir):
    rows = []
    with open(os.path.join(golden_dir, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers(golden_dir):
    for ctr, key, out in _kat(golden_dir):
        assert list(rng.philox4x32_10(ctr, key)) == out


def test_philox_vectorised_matches_scalar():
    r = np.random.default_rng(1)
    c = r.integers(0, 2**32, size=(4, 200), dtype=np.uint64)
    k0, k1 = 0x12345678, 0x9ABCDEF0
    vec = rng.philox4x32_10_np(c[0], c[1], c[2], c[3], k0, k1)
    for i in range(200):
        ref = rng.philox4x32_10([int(c[j, i]) for j in range(4)], (k0, k1))
        assert tuple(int(v[i]) for v in vec) == ref


def test_word_stream_layout():
    # w(q) = Philox(ctr=(q//4, 0, tag, 0), key=(seed lo, seed hi))[q % 4]
    seed, tag = (7 << 32) | 3, 5
    s = rng.WordStream(seed, tag)
    blk = rng.philox4x32_10((2, 0, tag, 0), (3, 7))
    assert [s.word(8 + i) for i in range(4)] == list(blk)


@pytest.mark.parametrize("s", [1, 2, 3, 5, 7, 10, 1000, 2**31 + 1, 2**32 - 1, 2**32])
def test_lemire_acceptance_region(s):
    """Counting argument: with t = 2^32 mod s, word x is accepted iff
    (x*s mod 2^32) >= t, and every output v in [0, s) then has exactly
    floor(2^32 / s) preimages.  Check the region boundaries of sampled v."""
    t = (2**32) % s
    per = 2**32 // s
    r = np.random.default_rng(s)
    vs = set([0, s - 1] + [int(v) for v in r.integers(0, s, size=20)])
    for v in vs:
        # accepted preimages of v: x with v*2^32 + t <= x*s < (v+1)*2^32
        lo = -(-(v * 2**32 + t) // s)
        hi = -(-((v + 1) * 2**32) // s)  # exclusive
        assert hi - lo == per
        for x in (lo, hi - 1):
            ok, val = rng.lemire_accept(x, s)
            assert ok and val == v
        if lo - 1 >= 0:
            ok, val = rng.lemire_accept(lo - 1, s)
            assert (not ok) or val == v - 1
        if hi < 2**32:
            ok, val = rng.lemire_accept(hi, s)
            assert (not ok) or val == v + 1


def test_floyd_spec_examples():
    assert list(rng.floyd(5, 5, 123, 1)) == [0, 1, 2, 3, 4]
    assert np.array_equal(rng.floyd(100, 10, 7, 1), rng.floyd(100, 10, 7, 1))
    with pytest.raises(ValueError):
        rng.floyd(4, 5, 0, 1)
    assert rng.floyd(10, 0, 0, 1).size == 0


def test_floyd_sorted_distinct_in_range():
    for seed in range(50):
        idx = rng.floyd(1000, 37, seed, 2)
        assert idx.dtype == np.int64
        assert np.all(np.diff(idx) > 0) and idx[0] >= 0 and idx[-1] < 1000


def test_floyd_index_frequency():
    # (100, 10, seeds 1..1000) -> each index frequency within 5 sigma of 0.1
    counts = np.zeros(100)
    for seed in range(1, 1001):
        counts[rng.floyd(100, 10, seed, 1)] += 1
    p = 0.1
    sigma = math.sqrt(1000 * p * (1 - p))
    assert np.all(np.abs(counts - 1000 * p) < 5 * sigma)


def test_floyd_uniform_over_subsets():
    # Floyd draws every k-subset with probability 1/C(N, k): chi-square over 10 subsets.
    from itertools import combinations
    subs = {c: 0 for c in combinations(range(5), 2)}
    T = 6000
    for seed in range(T):
        subs[tuple(int(v) for v in rng.floyd(5, 2, seed, 3))] += 1
    exp = T / len(subs)
    chi2 = sum((c - exp) ** 2 / exp for c in subs.values())
    assert chi2 < 33.7  # chi2(9) 99.99th percentile ~ 33.7


def test_tags_give_independent_streams():
    a = rng.floyd(10**6, 50, 0, rng.TAG_PILOT_ROWS)
    b = rng.floyd(10**6, 50, 0, rng.TAG_PILOT_COLS)
    assert not np.array_equal(a, b)
