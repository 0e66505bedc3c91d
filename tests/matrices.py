"""Test fixtures: small matrices restated from the reference's tests/oracles.hpp
and acceptance.cpp (TEST INFRASTRUCTURE). Random streams come from the oracle's
mt19937_64 so they match the reference fixtures draw for draw."""
from __future__ import annotations

import numpy as np

from paper_2409_11515_b200 import SparseMatrix


class MT:
    """Sequential mt19937_64 stream (draws fetched in blocks from the oracle)."""

    def __init__(self, oracle, seed: int, block: int = 1 << 16):
        self.o, self.seed, self.block = oracle, seed, block
        self.buf = oracle.mt_draws(seed, block)
        self.pos = 0

    def next(self) -> int:
        if self.pos >= self.buf.size:
            self.block *= 2
            self.buf = self.o.mt_draws(self.seed, self.block)
        v = int(self.buf[self.pos])
        self.pos += 1
        return v

    def uniform01(self) -> float:  # rng.hpp:31-33
        return float(self.next() >> 11) * 2.0 ** -53

    def uniform_in(self, lo, hi) -> float:  # rng.hpp:36-38
        return lo + (hi - lo) * self.uniform01()

    def normal(self) -> float:  # rng.hpp:61-65
        u1 = 1.0 - self.uniform01()
        u2 = self.uniform01()
        return float(np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2))


def random_sparse(oracle, n: int, density: float, seed: int) -> SparseMatrix:
    """oracles.hpp:168-179: nonzero diagonal in [0.5,1.5), off-diagonals U[-1,1)."""
    g = MT(oracle, seed)
    t = []
    for i in range(n):
        t.append((i, i, g.uniform_in(0.5, 1.5)))
        for j in range(n):
            if j == i:
                continue
            if g.uniform01() < density:
                t.append((i, j, g.uniform_in(-1.0, 1.0)))
    return SparseMatrix.from_triplets(n, n, t)


def diag_matrix(d) -> SparseMatrix:
    return SparseMatrix.from_triplets(len(d), len(d), [(i, i, float(v)) for i, v in enumerate(d)])


def laplacian2d(grid: int) -> SparseMatrix:
    """acceptance.cpp:240-254 (5-point, diagonal 4, Dirichlet)."""
    t = []
    idx = lambda r, c: r * grid + c  # noqa: E731
    for r in range(grid):
        for c in range(grid):
            t.append((idx(r, c), idx(r, c), 4.0))
            if r > 0:
                t.append((idx(r, c), idx(r - 1, c), -1.0))
            if r + 1 < grid:
                t.append((idx(r, c), idx(r + 1, c), -1.0))
            if c > 0:
                t.append((idx(r, c), idx(r, c - 1), -1.0))
            if c + 1 < grid:
                t.append((idx(r, c), idx(r, c + 1), -1.0))
    return SparseMatrix.from_triplets(grid * grid, grid * grid, t)


def row_scaled(a: SparseMatrix, oracle, seed: int, lo=-3.0, hi=3.0) -> SparseMatrix:
    """BASELINE config 1: each row scaled by 10^U(lo,hi) drawn row-major from mt19937_64(seed)."""
    u = oracle.uniform_in(seed, a.nrows, lo, hi)
    vals = a.values.copy()
    rp = a.row_offsets
    for i in range(a.nrows):
        vals[rp[i]:rp[i + 1]] *= 10.0 ** u[i]
    return SparseMatrix(a.nrows, a.ncols, rp, a.col_indices, vals)


def svd_constructed(n: int, sigmas, seed: int) -> tuple[SparseMatrix, np.ndarray]:
    """A = U diag(sigma) V^T with random orthogonal factors (oracles.hpp:155-164);
    the spectrum is known by construction."""
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    d = (u * np.asarray(sigmas)) @ v.T
    r, c = np.nonzero(d)
    return SparseMatrix.from_coo(n, n, r, c, d[r, c]), d


def geometric_sigmas(n: int, smax: float, kappa: float) -> np.ndarray:
    """oracles.hpp:132-145."""
    if n == 1:
        return np.array([smax])
    ratio = kappa ** (-1.0 / (n - 1))
    s, v = [], smax
    for _ in range(n):
        s.append(v)
        v *= ratio
    return np.array(s)


def cfg(**kw):
    from paper_2409_11515_b200 import AdamConfig
    return AdamConfig(**kw)
