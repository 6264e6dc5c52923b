"""Eigenpairs of complex Hermitian operators (configs 3 and 5) through the real embedding.

The reference solver is real symmetric only (``solve`` in proj/src/solver.cpp:119-360
takes a CsrMatrixd). For H = A + iB Hermitian, the real symmetric

    S = [[A, -B],
         [B,  A]]          (2n x 2n)

satisfies S [x; y] = lambda [x; y]  <=>  H (x + iy) = lambda (x + iy): every eigenvalue of H is an
eigenvalue of S with twice its multiplicity, and every eigenvector of S maps to one of H. This is the
same embedding that pins the complex filter to the real (reference-exact) one.

``solve_hermitian`` runs the GPU ``solve`` on S (the window [a, b] unchanged; the subspace size follows
the reference rule on S's doubled count, or twice ``p_override``), maps the converged S eigenvectors to
C^n, extracts an orthonormal basis of their span (each eigenvector of H arrives twice, as v and i v),
and finishes with one Rayleigh-Ritz step on H itself (the complex SpMM on the device), so the returned
eigenpairs are H's, with their residuals measured on H.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .operator import Context, DeviceCsr, maspmm
from .solver import SolveResult, SolverConfig, solve
from .sparse import CsrMatrix


def hermitian_embedding(h: CsrMatrix) -> CsrMatrix:
    """The real 2n x 2n embedding S of a complex Hermitian CSR matrix H (structural zeros dropped).

    Row r of S holds (c, Re h_rc) and (c + n, -Im h_rc); row r + n holds (c, Im h_rc) and
    (c + n, Re h_rc). Columns stay strictly ascending per row (all c < n <= c' + n).
    """
    if h.n_rows != h.n_cols:
        raise ValueError("hermitian_embedding: square matrices only")
    n = h.n_rows
    rp = np.asarray(h.row_ptr, np.int64)
    ci = np.asarray(h.col_idx, np.int64)
    v = np.asarray(h.values, np.complex128)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    re, im = v.real, v.imag
    blocks = [(rows, ci, re), (rows, ci + n, -im), (rows + n, ci, im), (rows + n, ci + n, re)]
    r = np.concatenate([b[0] for b in blocks])
    c = np.concatenate([b[1] for b in blocks])
    x = np.concatenate([b[2] for b in blocks])
    keep = x != 0.0
    return CsrMatrix.from_triplets(2 * n, 2 * n, r[keep], c[keep], x[keep])


def solve_hermitian(h: CsrMatrix, config: SolverConfig, ctx: Context | None = None) -> SolveResult:
    """Interior eigenpairs of a complex Hermitian CSR matrix in [interval_a, interval_b] (GPU)."""
    if not h.is_complex:
        raise ValueError("solve_hermitian: complex operator expected (use solve for real symmetric ones)")
    n = h.n_rows
    ctx = ctx or Context(0)
    ds = DeviceCsr(hermitian_embedding(h), ctx)
    cfg = dataclasses.replace(config, p_override=2 * config.p_override if config.p_override else None)
    r = solve(ds, cfg)
    ds.close()
    z = r.eigenvectors
    if z.shape[1] == 0:
        return dataclasses.replace(r, eigenvectors=np.zeros((n, 0), np.complex128))
    v = z[:n] + 1j * z[n:]
    # orthonormal basis of span(v): the Gram matrix of (v, i v) pairs has eigenvalues 2 and 0
    g = v.conj().T @ v
    d, w = np.linalg.eigh((g + g.conj().T) / 2)
    keep = d > 0.25 * float(d.max())
    u = v @ (w[:, keep] / np.sqrt(d[keep]))
    # one Rayleigh-Ritz step on H (complex SpMM on the device)
    dh = DeviceCsr(h, ctx)
    hu = maspmm(dh, u)
    t = u.conj().T @ hu
    theta, y = np.linalg.eigh((t + t.conj().T) / 2)
    vecs = u @ y
    hv = hu @ y
    res = np.linalg.norm(hv - vecs * theta, axis=0)
    dh.close()
    inside = (theta >= config.interval_a) & (theta <= config.interval_b)
    theta, vecs, res = theta[inside], vecs[:, inside], res[inside]
    return dataclasses.replace(r, eigenvalues=theta, eigenvectors=vecs,
                               max_residual=float(res.max()) if len(res) else 0.0)
