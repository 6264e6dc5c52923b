"""Synthetic operators of BASELINE.json's five configurations (seeded, vectorised numpy).

No dataset is involved: the reference paper measures on SuiteSparse DFT
Hamiltonians that are not available here; these seeded
generators with BASELINE.json's shapes and value distributions stand in for
them. Matrix randomness uses Philox streams >= 16 so it
never collides with the solver's streams 0-3 (philox.hpp:84-89).

Each generator returns a CsrMatrix with rows sorted by column (ascending), the
layout the kernel's accumulation order relies on.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .sparse import CsrMatrix, philox_gaussian, philox_uniform

STREAM_POTENTIAL = 16
STREAM_CENTRES = 17
STREAM_OFFBAND = 18


def _assemble(n: int, cols: np.ndarray, vals: np.ndarray, valid: np.ndarray) -> CsrMatrix:
    """Rows given as fixed-width candidate lists (already ascending per row) + validity mask."""
    counts = valid.sum(axis=1).astype(np.int64)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return CsrMatrix(n, n, row_ptr, np.ascontiguousarray(cols[valid], np.int64), np.ascontiguousarray(vals[valid]))


def stencil_3d(nx: int, offsets, weights, diag: np.ndarray) -> CsrMatrix:
    """Dirichlet stencil on an nx^3 grid (row = x + nx (y + nx z)); offsets in ascending linear order."""
    n = nx ** 3
    idx = np.arange(n, dtype=np.int64)
    x, y, z = idx % nx, (idx // nx) % nx, idx // (nx * nx)
    k = len(offsets)
    cols = np.empty((n, k), np.int64)
    vals = np.empty((n, k), np.float64)
    valid = np.empty((n, k), bool)
    for j, ((dx, dy, dz), w) in enumerate(zip(offsets, weights)):
        ok = (x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < nx) & (z + dz >= 0) & (z + dz < nx)
        cols[:, j] = idx + dx + nx * (dy + nx * dz)
        if (dx, dy, dz) == (0, 0, 0):
            vals[:, j] = diag
        else:
            vals[:, j] = w
        valid[:, j] = ok
    return _assemble(n, cols, vals, valid)


def _seven_point():
    offs = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    return offs, [-1.0] * 7


def _twenty_seven_point():
    """Compact 4th-order ("Mehrstellen") -Laplacian weights: 64/15, -7/15 (faces), -1/10 (edges), -1/30 (corners)."""
    offs, ws = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                m = abs(dx) + abs(dy) + abs(dz)
                offs.append((dx, dy, dz))
                ws.append({0: 64.0 / 15.0, 1: -7.0 / 15.0, 2: -1.0 / 10.0, 3: -1.0 / 30.0}[m])
    return offs, ws


def laplacian7_potential(nx: int, lo: float, hi: float, seed: int = 0) -> CsrMatrix:
    """7-point -Laplacian (diag 6, off -1) + diagonal potential uniform [lo, hi) (configs 1, 2)."""
    n = nx ** 3
    u = philox_uniform(seed, STREAM_POTENTIAL, 0, n)
    offs, ws = _seven_point()
    return stencil_3d(nx, offs, ws, 6.0 + (lo + (hi - lo) * u))


def dft_like_27pt(nx: int = 128, n_centres: int = 64, seed: int = 0) -> CsrMatrix:
    """27-point compact stencil + smooth Gaussian-sum local potential (config 4)."""
    n = nx ** 3
    cen = philox_uniform(seed, STREAM_CENTRES, 0, 3 * n_centres).reshape(n_centres, 3) * nx
    idx = np.arange(n, dtype=np.int64)
    pts = np.stack([idx % nx, (idx // nx) % nx, idx // (nx * nx)], axis=1).astype(np.float64)
    pot = np.zeros(n)
    width2 = (0.08 * nx) ** 2
    for c in cen:  # attractive wells of depth 2, width 8% of the box
        d2 = ((pts - c) ** 2).sum(axis=1)
        pot -= 2.0 * np.exp(-d2 / (2.0 * width2))
    offs, ws = _twenty_seven_point()
    return stencil_3d(nx, offs, ws, ws[13] + pot)


def peierls_lattice(L: int = 1000, phi: float = 1.0 / 64.0, seed: int = 0) -> CsrMatrix:
    """Complex Hermitian square-lattice tight binding with Landau-gauge Peierls phases (config 3).

    Row = x + L y; hopping -1 on x-bonds, -exp(+-i 2 pi phi x) on y-bonds, on-site uniform [-1, 1); open BC.
    """
    n = L * L
    idx = np.arange(n, dtype=np.int64)
    x, y = idx % L, idx // L
    onsite = -1.0 + 2.0 * philox_uniform(seed, STREAM_POTENTIAL, 0, n)
    ph = np.exp(2j * math.pi * phi * x)
    cols = np.stack([idx - L, idx - 1, idx, idx + 1, idx + L], axis=1)
    vals = np.stack([-np.conj(ph), -np.ones(n), onsite.astype(np.complex128), -np.ones(n), -ph], axis=1)
    valid = np.stack([y > 0, x > 0, np.ones(n, bool), x < L - 1, y < L - 1], axis=1)
    return _assemble(n, cols, vals, valid)


def random_banded_hermitian(n: int, half_band: int, offband: int, seed: int = 0) -> CsrMatrix:
    """Banded |i-j| <= half_band plus `offband` random off-band entries per row, Re/Im ~ N(0,1), H = (A + A^H)/2 (config 5)."""
    # upper triangle (band + random off-band positions folded to r < c), deduplicated, then mirrored
    # with the conjugate so H is exactly Hermitian; entries (a + conj(a'))/2 of two N(0,1)+iN(0,1)
    # draws have variance 1/2 per part, which is what the upper values are drawn with.
    rows, cols = [], []
    for d in range(0, half_band + 1):
        i = np.arange(0, n - d, dtype=np.int64)
        rows.append(i)
        cols.append(i + d)
    u = philox_uniform(seed, STREAM_OFFBAND, 0, n * offband)
    r_off = np.repeat(np.arange(n, dtype=np.int64), offband)
    c_off = np.minimum((u * n).astype(np.int64), n - 1)
    keep = np.abs(c_off - r_off) > half_band
    lo, hi = np.minimum(r_off[keep], c_off[keep]), np.maximum(r_off[keep], c_off[keep])
    rows.append(lo)
    cols.append(hi)
    key = np.unique(np.concatenate(rows) * n + np.concatenate(cols))
    r, c = key // n, key % n
    g = philox_gaussian(seed, STREAM_OFFBAND + 1, 0, 2 * len(r)) * np.sqrt(0.5)
    v = g[0::2] + 1j * g[1::2]
    v[r == c] = v[r == c].real
    off = r != c
    r2 = np.concatenate([r, c[off]])
    c2 = np.concatenate([c, r[off]])
    v2 = np.concatenate([v, np.conj(v[off])])
    return CsrMatrix.from_triplets(n, n, r2, c2, v2)


@dataclass
class Config:
    """One BASELINE.json configuration: operator, block size, window and spectral bounds."""

    name: str
    description: str
    q: int
    window: tuple  # [a, b]
    bounds: tuple  # enclosure of the spectrum used for the filter map
    dtype: str
    build: callable

    def operator(self) -> CsrMatrix:
        return self.build()


# Bounds: Gershgorin enclosures (a valid [lambda_min, lambda_max] for the
# filter map). Windows: C1 literal 0.40-0.45 of the range; C2 a centred window
# holding ~200 eigenvalues (width from the density of states at the band
# centre, checked with the device Hutchinson estimator -- DESIGN.md section 5).
CONFIGS = {
    "c1": Config("c1", "3D 7-pt Laplacian 40^3 + U[0,1) potential, q=64", 64,
                 (0.40 * 13.0, 0.45 * 13.0), (0.0, 13.0), "f64",
                 lambda: laplacian7_potential(40, 0.0, 1.0)),
    "c2": Config("c2", "3D 7-pt Laplacian 100^3 + Anderson U[-2,2] (W=4), q=256", 256,
                 (6.0 - 0.000769, 6.0 + 0.000769), (-2.0, 14.0), "f64",
                 lambda: laplacian7_potential(100, -2.0, 2.0)),
    "c3": Config("c3", "2D Peierls lattice 1000^2, phi=1/64, on-site U[-1,1], complex128, q=384", 384,
                 (-0.0005, 0.0005), (-5.0, 5.0), "c128",
                 lambda: peierls_lattice(1000)),
    # Config 1 for END-TO-END solves: the literal 0.40-0.45 window holds ~6,000 eigenvalues against block 64
    # (p >= e is violated); this window is centred at 0.425 of the range and narrowed to
    # ~35 eigenvalues, so the reference rule p = max(ceil(1.8 e), e + 5, 10) applies.
    "c1s": Config("c1s", "3D 7-pt Laplacian 40^3 + U[0,1) potential, solve window ~35 eigenvalues", 64,
                  (0.425 * 13.0 - 0.002, 0.425 * 13.0 + 0.002), (0.0, 13.0), "f64",
                  lambda: laplacian7_potential(40, 0.0, 1.0)),
    "c4": Config("c4", "3D 27-pt Mehrstellen 128^3 + Gaussian-sum potential, q=1024", 1024,
                 (0.30, 0.32), (-2.0, 8.6), "f64",
                 lambda: dft_like_27pt(128)),
    # Config 5 (n = 4e6, half-band 250, ~2.16 G nonzeros, complex128, q = 384) needs ~100 GB of host
    # memory just to assemble; c5s keeps its row structure (band 250 + 20 random off-band entries per
    # row, Re/Im ~ N(0, 1/2)) at n = 200,000 for tests and kernel measurements.
    "c5s": Config("c5s", "random banded Hermitian n=2e5, half-band 250 + 20 off-band/row, complex128, q=384", 384,
                  (-1.0, 1.0), (-60.0, 60.0), "c128",
                  lambda: random_banded_hermitian(200_000, 250, 20)),
}


def filter_degree(cfg: Config, c: float = 1.4) -> int:
    """initial_degree of the config's window (cheb_filter.cpp:181-187; solver.cpp:138-146)."""
    lmin, lmax = cfg.bounds
    span = lmax - lmin
    l1, l2 = 2.0 / span, -(lmax + lmin) / span
    mapc = lambda v: min(max(l1 * v + l2, -1.0), 1.0)  # noqa: E731
    alpha, beta = math.acos(mapc(cfg.window[0])), math.acos(mapc(cfg.window[1]))
    return max(int(math.ceil(c / (alpha - beta))) - 1, 1)
