"""Seeded synthetic inputs for the CABS hot path (shared by oracle-side tests and
the CUDA-side harness).

This module holds NO arithmetic of the method: it only builds the input matrix A
of each BASELINE.json config (recipes: DESIGN.md "Input recipe").
The paper's Table-1 datasets are not available; these seeded
synthetic matrices stand in for them.

Every random value is keyed by (seed, tag, 250-row chunk index), so the rows a
rank generates for its shard are bit-identical to the same rows of the globally
generated matrix on the same device type.  Factor products are
formed in float64 and rounded once to float32.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

CHUNK = 250


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    k1: int
    k2: int
    iters: int
    kind: str
    seed: int = 0
    note: str = ""


# BASELINE.json configs[0..4]; c5 is the implicit RBF source (make_rbf, never materialised).
CONFIGS = {
    "c1": Config("c1", 2000, 1500, 20, 20, 10, "gauss_factor_decay",
                 note="A = G1 diag(1/i) G2^T + 0.01 N, rank 20 (BASELINE configs[0])"),
    "c2": Config("c2", 20000, 10000, 50, 50, 20, "orth_decay",
                 note="A = U diag(i^-1.5) V^T + 1e-3 N, U,V orthonormal rank 200 (configs[1])"),
    "c3": Config("c3", 100000, 50000, 100, 100, 25, "clustered",
                 note="A_ij = <mu_c(i), nu_d(j)> + 0.05 N_ij, 64 Zipf(1.1) clusters/side (configs[2])"),
    "c4": Config("c4", 400000, 100000, 200, 200, 25, "gauss_factor",
                 note="A = G1 G2^T + 0.1 N, rank 500 (configs[3])"),
    "c5": Config("c5", 2000000, 1000000, 300, 300, 5, "rbf_mixture",
                 note="A_ij = exp(-|x_i - y_j|^2 / 2 sigma^2), x, y in R^16 from a 100-component "
                      "Gaussian mixture, sigma = median pairwise distance of 1e4 pairs (configs[4], Z23)"),
}

# the paper's sparse Table-1 shapes, synthetic sparse_lowrank stand-ins
# (a rank-r Gaussian-factor product with all but a `density` fraction of entries zeroed)
SPARSE_CONFIGS = {
    "s1": Config("s1", 27000, 46000, 100, 100, 25, "sparse_lowrank",
                 note="sparse_lowrank rank 20 at the movie-ratings shape and density 0.56% (Table 1, P:301)"),
    "s2": Config("s2", 18774, 61188, 100, 100, 25, "sparse_lowrank",
                 note="sparse_lowrank rank 20 at the newsgroup shape and density 0.22% (Table 1, P:302)"),
}
SPARSE_DENSITY = {"s1": 0.0056, "s2": 0.0022}
SPARSE_RANK = 20

RBF_DIM = 16
RBF_COMPONENTS = 100
RBF_SIGMA_PAIRS = 10000


def _gen(device, seed: int, tag: int, idx: int = 0) -> torch.Generator:
    g = torch.Generator(device=device)
    # splitmix-style key derivation; integer only
    x = (seed * 0x9E3779B97F4A7C15 + tag * 0xBF58476D1CE4E5B9 + idx * 0x94D049BB133111EB) & ((1 << 63) - 1)
    g.manual_seed(x)
    return g


def _randn(shape, device, seed, tag, idx=0, dtype=torch.float64):
    return torch.randn(shape, generator=_gen(device, seed, tag, idx), device=device, dtype=dtype)


def _zipf_labels(count, ncl, s, device, seed, tag, idx):
    p = torch.arange(1, ncl + 1, dtype=torch.float64, device=device) ** (-s)
    p = p / p.sum()
    return torch.multinomial(p, count, replacement=True, generator=_gen(device, seed, tag, idx))


class Generator:
    """Builds rows [r0, r1) of A for a config, chunk by chunk, on `device`."""

    def __init__(self, cfg: Config, device="cpu"):
        self.cfg = cfg
        self.device = torch.device(device)
        d, s = self.device, cfg.seed
        m, n = cfg.m, cfg.n
        if cfg.kind == "gauss_factor_decay":
            r = 20
            self.G2 = _randn((n, r), d, s, 17) * (1.0 / torch.arange(1, r + 1, dtype=torch.float64, device=d))
            self.noise = 0.01
        elif cfg.kind == "orth_decay":
            r = 200
            U, _ = torch.linalg.qr(_randn((m, r), d, s, 18))
            V, _ = torch.linalg.qr(_randn((n, r), d, s, 19))
            self.U = U
            self.G2 = V * (torch.arange(1, r + 1, dtype=torch.float64, device=d) ** -1.5)
            self.noise = 1e-3
        elif cfg.kind == "clustered":
            ncl, dim = 64, 100
            self.mu = _randn((ncl, dim), d, s, 20)
            nu = _randn((ncl, dim), d, s, 21)
            col_lab = torch.cat([_zipf_labels(min(CHUNK, n - c0), ncl, 1.1, d, s, 22, c0 // CHUNK)
                                 for c0 in range(0, n, CHUNK)])
            self.G2 = nu[col_lab]           # n x 100
            self.noise = 0.05
        elif cfg.kind == "gauss_factor":
            self.G2 = _randn((n, 500), d, s, 23)
            self.noise = 0.1  # variance 0.01 (Z22)
        else:
            raise ValueError(cfg.kind)

    def _left(self, c0, rows):
        cfg, d, s = self.cfg, self.device, self.cfg.seed
        ci = c0 // CHUNK
        if cfg.kind == "gauss_factor_decay":
            return _randn((rows, 20), d, s, 24, ci)
        if cfg.kind == "orth_decay":
            return self.U[c0:c0 + rows]
        if cfg.kind == "clustered":
            return self.mu[_zipf_labels(rows, 64, 1.1, d, s, 25, ci)]
        return _randn((rows, 500), d, s, 26, ci)

    def rows(self, r0: int, r1: int, out: torch.Tensor | None = None, lda: int | None = None):
        """float32 rows [r0, r1) (r0 a multiple of CHUNK), row-major with leading dim lda."""
        cfg = self.cfg
        n = cfg.n
        assert r0 % CHUNK == 0 or r0 == 0
        lda = lda or n
        if out is None:
            out = torch.empty((r1 - r0, lda), dtype=torch.float32, device=self.device)
        for c0 in range(r0, r1, CHUNK):
            rows = min(CHUNK, r1 - c0, cfg.m - c0)
            ci = c0 // CHUNK
            blk = self._left(c0, rows) @ self.G2.T
            blk += self.noise * _randn((rows, n), self.device, cfg.seed, 27, ci)
            out[c0 - r0:c0 - r0 + rows, :n] = blk.to(torch.float32)
        return out

    def full(self):
        return self.rows(0, self.cfg.m)


def make_A(name_or_cfg, device="cpu", r0=0, r1=None):
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    g = Generator(cfg, device)
    return g.rows(r0, cfg.m if r1 is None else r1)


def scaled(cfg: Config, m: int, n: int, k1: int | None = None, k2: int | None = None,
           iters: int | None = None, seed: int | None = None) -> Config:
    """Same recipe at another size (parity cases the oracle finishes in seconds)."""
    return Config(cfg.name + f"_{m}x{n}", m, n, k1 or cfg.k1, k2 or cfg.k2,
                  iters or cfg.iters, cfg.kind, cfg.seed if seed is None else seed, cfg.note)


def row_partition(m: int, rank: int, nranks: int, align: int = CHUNK):
    """Contiguous row block of rank (ceil split, aligned to generator chunks)."""
    per = int(math.ceil(m / nranks / align)) * align
    r0 = min(m, rank * per)
    r1 = min(m, r0 + per)
    return r0, r1


def col_partition(n: int, rank: int, nranks: int):
    per = int(math.ceil(n / nranks))
    c0 = min(n, rank * per)
    return c0, min(n, c0 + per)


def make_rbf(cfg: Config):
    """Inputs of the implicit RBF source (BASELINE.json configs[4]; reading Z23): x (m x 16) and
    y (n x 16) float32 on the CPU, independent draws from one mixture of 100 unit-covariance
    Gaussians with means 3 N(0, I_16) and equal weights; sigma = median (mean of the two middle
    order statistics) of |x_a - y_b| over 1e4 seeded pairs, in float64 on the float32 points.
    The matrix itself is never formed: both sides generate entries on access."""
    assert cfg.kind == "rbf_mixture"
    s = cfg.seed
    mu = 3.0 * _randn((RBF_COMPONENTS, RBF_DIM), "cpu", s, 30)

    def points(count, tag):
        comp = torch.randint(0, RBF_COMPONENTS, (count,), generator=_gen("cpu", s, tag))
        return (mu[comp] + _randn((count, RBF_DIM), "cpu", s, tag + 1)).to(torch.float32)

    x = points(cfg.m, 31)
    y = points(cfg.n, 33)
    a = torch.randint(0, cfg.m, (RBF_SIGMA_PAIRS,), generator=_gen("cpu", s, 35))
    b = torch.randint(0, cfg.n, (RBF_SIGMA_PAIRS,), generator=_gen("cpu", s, 36))
    dist = torch.sqrt(((x[a].double() - y[b].double()) ** 2).sum(1))
    ds = torch.sort(dist).values
    h = RBF_SIGMA_PAIRS // 2
    sigma = float(0.5 * (ds[h - 1] + ds[h]))
    return x, y, sigma


def make_sparse(cfg: Config, density: float, device="cpu", rank: int = SPARSE_RANK):
    """sparse_lowrank(m, n, r, density, seed): positions drawn per 250-row chunk (row i gets
    Binomial(n, density) uniform columns, duplicates merged), values (G1 G2^T)_ij / sqrt(r) of
    Gaussian factors at those positions (float64 products rounded once to float32).  Returns CSR
    (indptr int64[m+1], indices int32, values float32) on `device`, columns increasing per row."""
    d, s = torch.device(device), cfg.seed
    m, n = cfg.m, cfg.n
    G2 = _randn((n, rank), d, s, 40)
    rows_l, cols_l, vals_l = [], [], []
    for c0 in range(0, m, CHUNK):
        rows = min(CHUNK, m - c0)
        ci = c0 // CHUNK
        g = _gen(d, s, 41, ci)
        cnt = torch.binomial(torch.full((rows,), float(n), dtype=torch.float64, device=d),
                             torch.full((rows,), float(density), dtype=torch.float64, device=d), generator=g)
        cnt = cnt.to(torch.int64)
        r = torch.repeat_interleave(torch.arange(rows, device=d), cnt)
        c = torch.randint(0, n, (int(cnt.sum()),), generator=g, device=d)
        key = torch.unique(r * n + c)  # sorted: rows, then columns; duplicates merged
        r, c = key // n, key % n
        G1 = _randn((rows, rank), d, s, 42, ci)
        v = (G1[r] * G2[c]).sum(1) / math.sqrt(rank)
        rows_l.append(r + c0)
        cols_l.append(c)
        vals_l.append(v.to(torch.float32))
    r = torch.cat(rows_l)
    indptr = torch.zeros(m + 1, dtype=torch.int64, device=d)
    indptr[1:] = torch.cumsum(torch.bincount(r, minlength=m), 0)
    return indptr, torch.cat(cols_l).to(torch.int32), torch.cat(vals_l)


def csr_to_csc(indptr, indices, values, n):
    """The same matrix in compressed sparse column form (col_ptr int64[n+1], row_idx int32,
    values float32), rows increasing per column: a stable sort of the nonzeros by column."""
    m = indptr.numel() - 1
    rows = torch.repeat_interleave(torch.arange(m, device=indptr.device), indptr[1:] - indptr[:-1])
    order = torch.argsort(indices.to(torch.int64) * m + rows)
    col_ptr = torch.zeros(n + 1, dtype=torch.int64, device=indptr.device)
    col_ptr[1:] = torch.cumsum(torch.bincount(indices.to(torch.int64), minlength=n), 0)
    return col_ptr, rows[order].to(torch.int32), values[order]
