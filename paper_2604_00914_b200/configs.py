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

# The Philox4x32-10 draws behind the generators (sparse.philox_uniform / philox_gaussian, the
# library's restatement of philox.hpp). set_rng swaps in another implementation of the same
# streams -- bench.py's reference arm builds its operator with the CPU oracle's Philox so that
# arm never maps the product library; tests pin the two bitwise.
_RNG = {"uniform": None, "gaussian": None}


def set_rng(uniform=None, gaussian=None) -> None:
    """Use uniform(seed, stream, first, count) / gaussian(...) for matrix randomness (None: the library's)."""
    _RNG["uniform"], _RNG["gaussian"] = uniform, gaussian


def _uniform(seed, stream, first, count):
    return (_RNG["uniform"] or philox_uniform)(seed, stream, first, count)


def _gaussian(seed, stream, first, count):
    return (_RNG["gaussian"] or philox_gaussian)(seed, stream, first, count)


def _assemble(n: int, cols: np.ndarray, vals: np.ndarray, valid: np.ndarray) -> CsrMatrix:
    """Rows given as fixed-width candidate lists (already ascending per row) + validity mask."""
    counts = valid.sum(axis=1).astype(np.int64)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return CsrMatrix(n, n, row_ptr, np.ascontiguousarray(cols[valid], np.int64), np.ascontiguousarray(vals[valid]))


def stencil_3d(nx: int, offsets, weights, diag: np.ndarray, ny: int | None = None, nz: int | None = None) -> CsrMatrix:
    """Dirichlet stencil on an nx x ny x nz grid (default nx^3; row = x + nx (y + ny z)); offsets in
    ascending linear order."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64)
    x, y, z = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    k = len(offsets)
    cols = np.empty((n, k), np.int64)
    vals = np.empty((n, k), np.float64)
    valid = np.empty((n, k), bool)
    for j, ((dx, dy, dz), w) in enumerate(zip(offsets, weights)):
        ok = (x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < ny) & (z + dz >= 0) & (z + dz < nz)
        cols[:, j] = idx + dx + nx * (dy + ny * dz)
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
    u = _uniform(seed, STREAM_POTENTIAL, 0, n)
    offs, ws = _seven_point()
    return stencil_3d(nx, offs, ws, 6.0 + (lo + (hi - lo) * u))


def dft_like_27pt(nx: int = 128, n_centres: int = 64, seed: int = 0) -> CsrMatrix:
    """27-point compact stencil + smooth Gaussian-sum local potential (config 4)."""
    n = nx ** 3
    cen = _uniform(seed, STREAM_CENTRES, 0, 3 * n_centres).reshape(n_centres, 3) * nx
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
    onsite = -1.0 + 2.0 * _uniform(seed, STREAM_POTENTIAL, 0, n)
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
    u = _uniform(seed, STREAM_OFFBAND, 0, n * offband)
    r_off = np.repeat(np.arange(n, dtype=np.int64), offband)
    c_off = np.minimum((u * n).astype(np.int64), n - 1)
    keep = np.abs(c_off - r_off) > half_band
    lo, hi = np.minimum(r_off[keep], c_off[keep]), np.maximum(r_off[keep], c_off[keep])
    rows.append(lo)
    cols.append(hi)
    key = np.unique(np.concatenate(rows) * n + np.concatenate(cols))
    r, c = key // n, key % n
    g = _gaussian(seed, STREAM_OFFBAND + 1, 0, 2 * len(r)) * np.sqrt(0.5)
    v = g[0::2] + 1j * g[1::2]
    v[r == c] = v[r == c].real
    off = r != c
    r2 = np.concatenate([r, c[off]])
    c2 = np.concatenate([c, r[off]])
    v2 = np.concatenate([v, np.conj(v[off])])
    return CsrMatrix.from_triplets(n, n, r2, c2, v2)


def random_banded_hermitian_device(n: int, half_band: int, offband: int, seed: int = 0, chunk_rows: int = 65536,
                                   device: str = "cuda"):
    """Config 5 at full size, generated ON THE GPU: (row_ptr int64, col_idx int32, values complex128) CUDA tensors.

    Same structure and distribution as random_banded_hermitian (band |i-j| <= half_band plus `offband` random
    draws per row folded to the upper triangle and deduplicated, upper values Re/Im ~ N(0, 1/2), real diagonal,
    lower triangle the exact conjugate), but the n = 4e6 operator (2.16 G nonzeros, 43 GB) is never assembled
    on the host: the draws come from torch's seeded CUDA generator (not the Philox streams of the host generator,
    so the values differ from random_banded_hermitian's at equal n) and each row is laid out as
    [lower off-band | band | upper off-band], which is ascending column order without a sort of the band.
    """
    import torch

    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(0x5EED0000 + seed)
    hb = half_band
    # off-band pairs (lo, hi), lo < hi - hb, unique and sorted by (lo, hi)
    u = torch.rand(n * offband, generator=g, dtype=torch.float64, device=dev)
    c = torch.clamp((u * n).to(torch.int64), max=n - 1)
    del u
    r = torch.arange(n, device=dev, dtype=torch.int64).repeat_interleave(offband)
    keep = (c - r).abs() > hb
    key = torch.unique(torch.minimum(r[keep], c[keep]) * n + torch.maximum(r[keep], c[keep]))
    del r, c, keep
    lo, hi = key // n, key % n
    m = lo.numel()
    vo = torch.complex(torch.randn(m, generator=g, dtype=torch.float64, device=dev),
                       torch.randn(m, generator=g, dtype=torch.float64, device=dev)) * math.sqrt(0.5)
    # upper band values U[r, d] = H[r, r + d] (d = 0 real)
    ub = torch.complex(torch.randn(n, hb + 1, generator=g, dtype=torch.float64, device=dev),
                       torch.randn(n, hb + 1, generator=g, dtype=torch.float64, device=dev)) * math.sqrt(0.5)
    ub[:, 0] = ub[:, 0].real.to(torch.complex128)
    rows = torch.arange(n, device=dev, dtype=torch.int64)
    n_lo_off = torch.bincount(hi, minlength=n)  # row hi holds (hi, lo) left of its band
    n_hi_off = torch.bincount(lo, minlength=n)  # row lo holds (lo, hi) right of its band
    b_lo = torch.clamp(rows, max=hb)
    b_hi = torch.clamp(n - 1 - rows, max=hb)
    row_len = n_lo_off + b_lo + 1 + b_hi + n_hi_off
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(row_len, 0, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=torch.complex128, device=dev)
    band_start = row_ptr[:-1] + n_lo_off
    offs = torch.arange(-hb, hb + 1, device=dev, dtype=torch.int64)
    for r0 in range(0, n, chunk_rows):
        rr = rows[r0:r0 + chunk_rows, None]
        cc = rr + offs[None, :]
        ok = (cc >= 0) & (cc < n)
        pos = band_start[r0:r0 + chunk_rows, None] + offs[None, :] + b_lo[r0:r0 + chunk_rows, None]
        up = offs >= 0
        v = torch.empty(cc.shape, dtype=torch.complex128, device=dev)
        v[:, up] = ub[r0:r0 + chunk_rows]
        # lower band H[r, r - k] = conj(U[r - k, k]), k = 1..hb
        src_r = (rr + offs[None, ~up]).clamp(min=0)
        v[:, ~up] = ub[src_r, (-offs[~up])[None, :].expand_as(src_r)].conj()
        col[pos[ok]] = cc[ok].to(torch.int32)
        val[pos[ok]] = v[ok]
    del ub
    # upper off-band entries of row lo: after the band, in hi order (key order)
    first_lo = torch.searchsorted(lo, lo, right=False)
    p_up = band_start[lo] + b_lo[lo] + 1 + b_hi[lo] + (torch.arange(m, device=dev) - first_lo)
    col[p_up] = hi.to(torch.int32)
    val[p_up] = vo
    # lower off-band entries of row hi: first in the row, in lo order
    order = torch.argsort(hi * n + lo)
    hs, ls = hi[order], lo[order]
    first_hi = torch.searchsorted(hs, hs, right=False)
    p_dn = row_ptr[hs] + (torch.arange(m, device=dev) - first_hi)
    col[p_dn] = ls.to(torch.int32)
    val[p_dn] = vo[order].conj()
    return row_ptr, col, val


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
    device_build: callable | None = None  # GPU generator returning (row_ptr, col_idx, values) CUDA tensors

    def operator(self) -> CsrMatrix:
        return self.build()

    def device_operator(self, ctx=None):
        """The operator as a DeviceCsr, generated on the GPU when the config has a device generator."""
        from .operator import DeviceCsr

        if self.device_build is None:
            return DeviceCsr(self.operator(), ctx)
        import torch

        rp, ci, v = self.device_build()
        da = DeviceCsr.from_device(len(rp) - 1, len(rp) - 1, rp, ci, v, ctx)
        del rp, ci, v
        torch.cuda.empty_cache()
        return da


def _c5_host_unavailable():
    raise MemoryError("config c5 (n = 4e6, 2.16 G nonzeros) is generated on the GPU: use Config.device_operator()")


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
    # A SMALL replica of config 1 for the bench's measured CPU-vs-GPU solve: 16^3 grid, same potential
    # distribution, window of ~24 eigenvalues at 0.425 of the range (the CPU solver oracle takes ~10 s on
    # 8 host threads; c1s takes ~15 min there).
    "c1t": Config("c1t", "3D 7-pt Laplacian 16^3 + U[0,1) potential, solve window ~24 eigenvalues", 64,
                  (0.425 * 13.0 - 0.02, 0.425 * 13.0 + 0.02), (0.0, 13.0), "f64",
                  lambda: laplacian7_potential(16, 0.0, 1.0)),
    # bounds: the Gershgorin enclosure [-5.885, 8.533] (the 64 wells of depth 2 overlap down to -5.9;
    # Lanczos: [-5.47, 6.16]). An earlier (-2.0, 8.6) missed the wells' bottom: the filter diverged at
    # high degree (the trace estimate at k_max = 765 returned NaN); low-degree timings were unaffected.
    "c4": Config("c4", "3D 27-pt Mehrstellen 128^3 + Gaussian-sum potential, q=1024", 1024,
                 (0.30, 0.32), (-5.9, 8.6), "f64",
                 lambda: dft_like_27pt(128)),
    # Config 4 for an END-TO-END solve on ONE GPU: "~1000 eigenpairs, block 1024" needs p = 1.8 e ~ 1840
    # columns by the reference rule (six 2.1M x 1840 fp64 blocks = 185 GB, more than one B200 holds; the
    # row-sharded 8-GPU layout is the configuration's own answer). This window holds ~510 eigenvalues
    # (trace estimate: 851 in [0.30, 0.31]), so p ~ 920 fits one GPU.
    "c4w": Config("c4w", "3D 27-pt Mehrstellen 128^3 + Gaussian-sum potential, solve window ~510 eigenvalues", 1024,
                  (0.300, 0.306), (-5.9, 8.6), "f64",
                  lambda: dft_like_27pt(128)),
    # Config 5 (n = 4e6, half-band 250, ~2.16 G nonzeros, complex128, q = 384) needs ~100 GB of host
    # memory just to assemble; c5s keeps its row structure (band 250 + 20 random off-band entries per
    # row, Re/Im ~ N(0, 1/2)) at n = 200,000 for tests and kernel measurements.
    "c5s": Config("c5s", "random banded Hermitian n=2e5, half-band 250 + 20 off-band/row, complex128, q=384", 384,
                  (-1.0, 1.0), (-60.0, 60.0), "c128",
                  lambda: random_banded_hermitian(200_000, 250, 20)),
    # Config 5 at full size, generated on the GPU (random_banded_hermitian_device); one spectrum slice of
    # ~256 eigenvalues at the band centre: the semicircle density of a 541-nonzero/row unit-variance
    # Hermitian matrix, 2n/(pi R) with R = 2 sqrt(541) = 46.5, gives 54.8k eigenvalues per unit -> width
    # 0.0047. Bounds: the c5s enclosure [-60, 60] (same row statistics; checked by Lanczos in tools/c5_full.py).
    "c5": Config("c5", "random banded Hermitian n=4e6, half-band 250 + 20 off-band/row, complex128, q=384", 384,
                 (-0.00234, 0.00234), (-60.0, 60.0), "c128", _c5_host_unavailable,
                 lambda: random_banded_hermitian_device(4_000_000, 250, 20)),
}


def filter_degree(cfg: Config, c: float = 1.4) -> int:
    """initial_degree of the config's window (cheb_filter.cpp:181-187; solver.cpp:138-146)."""
    lmin, lmax = cfg.bounds
    span = lmax - lmin
    l1, l2 = 2.0 / span, -(lmax + lmin) / span
    mapc = lambda v: min(max(l1 * v + l2, -1.0), 1.0)  # noqa: E731
    alpha, beta = math.acos(mapc(cfg.window[0])), math.acos(mapc(cfg.window[1]))
    return max(int(math.ceil(c / (alpha - beta))) - 1, 1)
