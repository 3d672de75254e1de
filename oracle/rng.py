"""Counter-based RNG of the method, oracle side (TEST INFRASTRUCTURE ONLY).

Implements, from the written specification (SURVEY.md §8(c)
Z17), the randomness that Algorithm 2 step 1 needs: "randomly select k columns
and k rows" (Alg. 2 step 1) -- uniform sampling without
replacement, deterministic per seed.

* Philox4x32-10 (Salmon et al., SC'11), key = (seed mod 2^32, seed >> 32).
* Sequential word stream w(q) = Philox(ctr=(b mod 2^32, b >> 32, tag, 0))[q mod 4]
  with b = floor(q / 4).
* Lemire multiply-shift bounded integer in [0, s) with rejection.
* Floyd's algorithm for k distinct values in [0, N), output sorted ascending.

Everything is integer arithmetic on Python ints (or numpy uint64), so the GPU
implementation must agree bit for bit.  Shares no code with the CUDA path.
"""
from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF
PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85

# Tags (SURVEY.md §8(c) Z17 / DESIGN.md "RNG").
TAG_PILOT_ROWS = 1
TAG_PILOT_COLS = 2
TAG_INIT_ROWS = 3
TAG_INIT_COLS = 4
TAG_RESIDUAL_PAIRS = 5
TAG_LEVERAGE_ROWS = 6
TAG_LEVERAGE_COLS = 7
TAG_TARGET_ROWS = 8    # Sketch-CUR target sampling
TAG_TARGET_COLS = 9
TAG_HOLDOUT_ROWS = 10  # validation block of the rank sweep
TAG_HOLDOUT_COLS = 11


def philox4x32_10(ctr, key):
    """One Philox4x32-10 block: 4 x uint32 counter, 2 x uint32 key -> 4 x uint32."""
    c0, c1, c2, c3 = (int(x) & M32 for x in ctr)
    k0, k1 = (int(x) & M32 for x in key)
    for rnd in range(10):
        p0 = PHILOX_M0 * c0
        p1 = PHILOX_M1 * c2
        hi0, lo0 = p0 >> 32, p0 & M32
        hi1, lo1 = p1 >> 32, p1 & M32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & M32, lo1, (hi0 ^ c3 ^ k1) & M32, lo0
        if rnd != 9:
            k0 = (k0 + PHILOX_W0) & M32
            k1 = (k1 + PHILOX_W1) & M32
    return (c0, c1, c2, c3)


def philox4x32_10_np(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 over numpy arrays of counters (uint64 holding uint32)."""
    c0 = np.asarray(c0, dtype=np.uint64) & np.uint64(M32)
    c1 = np.asarray(c1, dtype=np.uint64) & np.uint64(M32)
    c2 = np.asarray(c2, dtype=np.uint64) & np.uint64(M32)
    c3 = np.asarray(c3, dtype=np.uint64) & np.uint64(M32)
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 = np.uint64(int(k0) & M32)
    k1 = np.uint64(int(k1) & M32)
    m0, m1 = np.uint64(PHILOX_M0), np.uint64(PHILOX_M1)
    mask, sh = np.uint64(M32), np.uint64(32)
    for rnd in range(10):
        p0 = m0 * c0  # < 2^64, exact in uint64
        p1 = m1 * c2
        hi0, lo0 = p0 >> sh, p0 & mask
        hi1, lo1 = p1 >> sh, p1 & mask
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & mask, lo1, (hi0 ^ c3 ^ k1) & mask, lo0
        if rnd != 9:
            k0 = np.uint64((int(k0) + PHILOX_W0) & M32)
            k1 = np.uint64((int(k1) + PHILOX_W1) & M32)
    return c0, c1, c2, c3


def seed_key(seed: int):
    seed = int(seed) & ((1 << 64) - 1)
    return (seed & M32, seed >> 32)


class WordStream:
    """Sequential consumer of 32-bit words w(0), w(1), ... for (seed, tag)."""

    def __init__(self, seed: int, tag: int):
        self.key = seed_key(seed)
        self.tag = int(tag) & M32
        self.q = 0
        self._block = None
        self._block_id = -1

    def word(self, q: int) -> int:
        b = q // 4
        if b != self._block_id:
            self._block = philox4x32_10((b & M32, (b >> 32) & M32, self.tag, 0), self.key)
            self._block_id = b
        return self._block[q % 4]

    def next(self) -> int:
        w = self.word(self.q)
        self.q += 1
        return w


def lemire_accept(x: int, s: int):
    """Lemire multiply-shift step: returns (accepted, value) for word x and bound s."""
    m = x * s
    lo = m & M32
    if lo < s:
        thresh = ((1 << 32) - s) % s
        if lo < thresh:
            return False, None
    return True, m >> 32


def bounded(stream: WordStream, s: int) -> int:
    """Uniform integer in [0, s), 1 <= s <= 2^32, drawing more words on rejection."""
    if not (1 <= s <= (1 << 32)):
        raise ValueError("bound out of range")
    while True:
        ok, v = lemire_accept(stream.next(), s)
        if ok:
            return v


def floyd(N: int, k: int, seed: int, tag: int) -> np.ndarray:
    """k distinct indices uniform in [0, N) (Floyd), sorted ascending, int64.

    P:195 "randomly select k columns and k rows"; S:137-141 (k > N is an error).
    """
    if k < 0 or k > N:
        raise ValueError(f"cannot draw k={k} distinct indices from N={N}")
    stream = WordStream(seed, tag)
    chosen = set()
    for j in range(N - k, N):
        t = bounded(stream, j + 1)
        chosen.add(j if t in chosen else t)
    return np.array(sorted(chosen), dtype=np.int64)


def uniform01(seed: int, tag: int, idx) -> np.ndarray:
    """Per-point uniform in (0, 1): Philox block of counter
    (idx mod 2^32, idx >> 32, tag, 1) -> words w0, w1; u = ((w0 >> 5) 2^26 + (w1 >> 6) + 1/2) 2^-53
    (53 random bits, exact in float64, never 0 or 1).  Counter word 3 = 1 keeps these blocks
    apart from the sequential word stream (word 3 = 0)."""
    idx = np.asarray(idx, dtype=np.uint64)
    k0, k1 = seed_key(seed)
    w0, w1, _, _ = philox4x32_10_np(idx & np.uint64(M32), idx >> np.uint64(32), np.uint64(int(tag) & M32),
                                     np.uint64(1), k0, k1)
    a = (w0 >> np.uint64(5)).astype(np.float64)
    b = (w1 >> np.uint64(6)).astype(np.float64)
    return (a * 67108864.0 + b + 0.5) * 2.0 ** -53


def _lemire_np(x, s):
    """Vectorised Lemire step: (accepted mask, value) for uint64 arrays of 32-bit words x."""
    s64 = np.uint64(s)
    prod = x * s64  # x < 2^32, s <= 2^32: exact in uint64
    lo = prod & np.uint64(M32)
    thresh = np.uint64(((1 << 32) - s) % s)
    return lo >= thresh, prod >> np.uint64(32)


def residual_pairs(seed: int, T: int, m: int, n: int, t0: int = 0):
    """T i.i.d. uniform entry positions (i, j) in [0, m) x [0, n) for the sampled residual
    (SURVEY.md Z17 / Z23 "uniform subset" = pairs with replacement).

    Pair t (t = t0 .. t0+T-1) reads Philox blocks of counter (t mod 2^32, t >> 32, 5, a) for
    attempts a = 0, 1, ...: i = Lemire(word 0, m), on rejection Lemire(word 1, m), then the
    next attempt's words 0, 1; j likewise from words 2, 3.  Returns int64 arrays (i, j)."""
    if not (1 <= m <= (1 << 32)) or not (1 <= n <= (1 << 32)):
        raise ValueError("bounds out of range")
    t = np.arange(t0, t0 + T, dtype=np.uint64)
    k0, k1 = seed_key(seed)
    out = []
    for s, (wa, wb) in ((m, (0, 1)), (n, (2, 3))):
        val = np.zeros(T, dtype=np.uint64)
        todo = np.arange(T)
        a = 0
        while todo.size:
            tt = t[todo]
            words = philox4x32_10_np(tt & np.uint64(M32), tt >> np.uint64(32), np.uint64(TAG_RESIDUAL_PAIRS),
                                     np.uint64(a), k0, k1)
            ok0, v0 = _lemire_np(words[wa], s)
            ok1, v1 = _lemire_np(words[wb], s)
            done = ok0 | ok1
            val[todo[done]] = np.where(ok0, v0, v1)[done]
            todo = todo[~done]
            a += 1
        out.append(val.astype(np.int64))
    return out[0], out[1]
